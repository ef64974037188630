// geometry.cuh -- device-side addressing for the three tilings (CellIndex, CellCenter,
// Children/Parent/Neighbors), PAPER.md sections 4-6.
//
// Bit-exactness contract (D11/D12): keys and centres follow fixed IEEE-754
// binary64 expression sequences with explicit __d*_rn intrinsics, so no FMA contraction
// can change a rounding.  The septree uses integer lattice arithmetic (App. B.1 of
// SURVEY: multiplication by lambda = 2 + i sqrt3 and digit extraction), the triangle-
// quadtree the level-by-level descent of P:358-364 and Table 1, the
// quadtree Morton order.
#pragma once
#include <stdint.h>

#define FMM_S3 1.7320508075688772  // sqrt(3) rounded to binary64
#define FMM_H 0.8660254037844386   // sqrt(3)/2 rounded to binary64

struct DGeo {
  int tiling, L, B;
  int64_t K;
  double root_x, root_y, root_size;
  double sept_A, sept_Bc, sept_D3r;  // 1.5 r, 0.5 (S3 r), 3 r
};

__host__ __device__ inline int64_t ipow_d(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// ------------------------------------------------------------------ quadtree (Morton, D7)
__host__ __device__ inline uint32_t spread2(uint32_t v) {  // interleave zeros: bit b -> bit 2b
  v &= 0x0000ffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__host__ __device__ inline uint32_t compact2(uint32_t v) {
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0f0f0f0fu;
  v = (v | (v >> 4)) & 0x00ff00ffu;
  v = (v | (v >> 8)) & 0x0000ffffu;
  return v;
}

__device__ inline bool quad_key(const DGeo& g, double x, double y, uint32_t* key) {
  double fx = __ddiv_rn(__dsub_rn(x, g.root_x), g.root_size);
  double fy = __ddiv_rn(__dsub_rn(y, g.root_y), g.root_size);
  if (!(fx >= 0.0 && fx <= 1.0 && fy >= 0.0 && fy <= 1.0)) return false;
  int64_t side = (int64_t)1 << g.L;
  int64_t i = (int64_t)floor(ldexp(fx, g.L)), j = (int64_t)floor(ldexp(fy, g.L));
  if (i == side) i = side - 1;
  if (j == side) j = side - 1;
  *key = spread2((uint32_t)i) | (spread2((uint32_t)j) << 1);
  return true;
}

__device__ inline double2 quad_centre(const DGeo& g, int l, int64_t n) {
  uint32_t i = compact2((uint32_t)n), j = compact2((uint32_t)(n >> 1));
  double S = g.root_size;
  double cx = __dadd_rn(g.root_x, __dmul_rn(S, ldexp((double)(2 * (int64_t)i + 1), -(l + 1))));
  double cy = __dadd_rn(g.root_y, __dmul_rn(S, ldexp((double)(2 * (int64_t)j + 1), -(l + 1))));
  return make_double2(cx, cy);
}

__device__ inline int quad_neighbors(int l, int64_t n, int64_t* out) {
  int64_t i = compact2((uint32_t)n), j = compact2((uint32_t)(n >> 1)), side = (int64_t)1 << l;
  int c = 0;
  for (int dj = -1; dj <= 1; ++dj)
    for (int di = -1; di <= 1; ++di) {
      if (!di && !dj) continue;
      int64_t a = i + di, b = j + dj;
      if (a < 0 || b < 0 || a >= side || b >= side) continue;
      out[c++] = (int64_t)(spread2((uint32_t)a) | (spread2((uint32_t)b) << 1));
    }
  return c;
}

// ------------------------------------------------------------------ septree (integer lattice)
// unit digit d -> lattice step on the (digit-1 at 30 deg, digit-2 at 90 deg) basis (D3, D5)
//   UB = {0, 1, 0, -1, -1, 0, 1}, UC = {0, 0, 1, 1, 0, -1, -1}, packed as 2-bit (v + 1) fields
__host__ __device__ inline void sept_unit(int d, int64_t* b, int64_t* c) {
  *b = (int64_t)((0x2419u >> (2 * d)) & 3u) - 1;
  *c = (int64_t)((0x1a5u >> (2 * d)) & 3u) - 1;
}
// address (l digits, MSB first) -> lattice coordinates of the level-l lattice: Horner with
// lambda, v <- M v + unit(t_i), M(b, c) = (b - 2c, 2b + 3c)
__host__ __device__ inline void sept_addr_to_lattice(int64_t n, int l, int64_t* b, int64_t* c) {
  // digits LSB first by constant division (n < 7^10 < 2^32), packed 3 bits each, then Horner
  // from the most significant digit
  uint32_t m = (uint32_t)n;
  uint64_t packed = 0;
  for (int i = 0; i < l; ++i) {
    packed |= (uint64_t)(m % 7u) << (3 * i);
    m /= 7u;
  }
  int64_t B = 0, C = 0;
  for (int i = l - 1; i >= 0; --i) {
    const int d = (int)((packed >> (3 * i)) & 7u);
    int64_t nb = B - 2 * C, nc = 2 * B + 3 * C;
    int64_t ub, uc;
    sept_unit(d, &ub, &uc);
    B = nb + ub;
    C = nc + uc;
  }
  *b = B;
  *c = C;
}
// apply M k times (zero-extension by k digits)
__host__ __device__ inline void sept_lambda_pow(int k, int64_t* b, int64_t* c) {
  for (int i = 0; i < k; ++i) {
    int64_t nb = *b - 2 * *c, nc = 2 * *b + 3 * *c;
    *b = nb;
    *c = nc;
  }
}
// lattice -> address with at most maxd digits (false if more are needed): digit extraction
// d = T[(b + 3c) mod 7], (b, c) <- M^-1((b, c) - unit(d)), M^-1 = [[3, 2], [-2, 1]] / 7
__host__ __device__ inline bool sept_lattice_to_addr(int64_t b64, int64_t c64, int maxd, int64_t* n) {
  // an address of <= 10 digits has |b|, |c| < 7^5 * 3 (far below 2^27): larger lattice
  // points are out of the domain, and the rest fits 32-bit arithmetic (exact /7 by the
  // modular inverse 0xB6DB6DB7 of 7 mod 2^32, since the differences below are multiples of 7)
  if (b64 <= -(1 << 27) || b64 >= (1 << 27) || c64 <= -(1 << 27) || c64 >= (1 << 27)) return false;
  // T = {0, 1, 3, 2, 5, 6, 4} as nibbles (no local-memory table)
  constexpr uint32_t T = 0x4652310u;
  int32_t b = (int32_t)b64, c = (int32_t)c64;
  int64_t key = 0, pw = 1;
  for (int k = 0; k < maxd; ++k) {
    if (b == 0 && c == 0) break;
    int r = (b + 3 * c) % 7;
    if (r < 0) r += 7;
    const int d = (int)((T >> (4 * r)) & 7u);
    int64_t ub, uc;
    sept_unit(d, &ub, &uc);
    b -= (int32_t)ub;
    c -= (int32_t)uc;
    const int32_t nb = (int32_t)((uint32_t)(3 * b + 2 * c) * 0xB6DB6DB7u);
    const int32_t nc = (int32_t)((uint32_t)(-2 * b + c) * 0xB6DB6DB7u);
    b = nb;
    c = nc;
    key += d * pw;
    pw *= 7;
  }
  if (b != 0 || c != 0) return false;
  *n = key;
  return true;
}

__device__ inline bool sept_key(const DGeo& g, double x, double y, uint32_t* key) {
  double xp = __dsub_rn(x, g.root_x), yp = __dsub_rn(y, g.root_y);
  double b = __ddiv_rn(__dmul_rn(2.0, xp), g.sept_D3r);                  // eq. P:212
  double c = __ddiv_rn(__dsub_rn(__dmul_rn(yp, FMM_S3), xp), g.sept_D3r);
  if (!(fabs(b) < 1.0e9) || !(fabs(c) < 1.0e9)) return false;
  const double bf = floor(b), bc = ceil(b), cf = floor(c), cc = ceil(c);  // eq. P:237 order
  double bb = bf, bcc = cf, bestd = 0.0;  // best candidate (first wins ties)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double qb = (q & 1) ? bc : bf, qc = (q & 2) ? cc : cf;  // (bf,cf) (bc,cf) (bf,cc) (bc,cc)
    double lx = __dmul_rn(g.sept_A, qb);                                  // eq. P:230
    double ly = __dmul_rn(g.sept_Bc, __dadd_rn(__dmul_rn(2.0, qc), qb));
    double dx = __dsub_rn(xp, lx), dy = __dsub_rn(yp, ly);
    double d = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    if (q == 0 || d < bestd) {
      bb = qb;
      bcc = qc;
      bestd = d;
    }
  }
  int64_t n;
  if (!sept_lattice_to_addr((int64_t)bb, (int64_t)bcc, g.L, &n)) return false;
  *key = (uint32_t)n;
  return true;
}

__device__ inline double2 sept_centre(const DGeo& g, int l, int64_t n) {
  int64_t b, c;
  sept_addr_to_lattice(n, l, &b, &c);
  sept_lambda_pow(g.L - l, &b, &c);  // zero-extend to the leaf lattice
  double cx = __dadd_rn(__dmul_rn(g.sept_A, (double)b), g.root_x);
  double cy = __dadd_rn(__dmul_rn(g.sept_Bc, (double)(2 * c + b)), g.root_y);
  return make_double2(cx, cy);
}

// Neighbors(n, l) = n (*) {1..6} kept if < 7^l, as lattice additions
__device__ inline int sept_neighbors(int l, int64_t n, int64_t* out) {
  int64_t b, c;
  sept_addr_to_lattice(n, l, &b, &c);
  int cnt = 0;
  for (int d = 1; d <= 6; ++d) {
    int64_t ub, uc, a;
    sept_unit(d, &ub, &uc);
    if (sept_lattice_to_addr(b + ub, c + uc, l, &a)) out[cnt++] = a;
  }
  return cnt;
}

// ------------------------------------------------------------------ triangle-quadtree
__device__ inline bool triq_key(const DGeo& g, double x, double y, uint32_t* key) {
  double xp = __dsub_rn(x, g.root_x), yp = __dsub_rn(y, g.root_y);
  double R0 = g.root_size, eps = __dmul_rn(1e-12, R0), lim = __dadd_rn(R0, eps);
  // closed root triangle with a 1e-12 R0 slack (D11)
  if (!(yp >= __dsub_rn(-0.5 * R0, eps)) || !(__dadd_rn(__dmul_rn(FMM_S3, xp), yp) <= lim) ||
      !(__dadd_rn(__dmul_rn(-FMM_S3, xp), yp) <= lim))
    return false;
  double u = 0.0, v = 0.0;
  double up = 1.0;
  uint32_t t = 0;
  double Ri = R0;
  for (int i = 1; i <= g.L; ++i) {
    Ri = 0.5 * Ri;  // = R0 2^-i exactly (as ldexp)
    double RH = __dmul_rn(Ri, FMM_H), half = 0.5 * Ri;
    double su = up * Ri, sh = up * half;  // exact
    const double vs = __dsub_rn(v, sh);
    int best = 0;
    double bestd = 0.0, bu = u, bv = v;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double cu = q < 2 ? u : (q == 2 ? __dsub_rn(u, RH) : __dadd_rn(u, RH));
      const double cv = q == 0 ? v : (q == 1 ? __dadd_rn(v, su) : vs);
      double dx = __dsub_rn(xp, cu), dy = __dsub_rn(yp, cv);
      double d = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      if (q == 0 || d < bestd) {
        best = q;
        bestd = d;
        bu = cu;
        bv = cv;
      }
    }
    u = bu;
    v = bv;
    if (best == 0) up = -up;  // centre child: orientation flips
    t = t * 4 + best;
  }
  *key = t;
  return true;
}

// running sum of the child offsets (P:326-333 with exact cos/sin, D12); s flips after a 0 digit
__device__ inline double2 triq_centre(const DGeo& g, int l, int64_t n) {
  double u = 0.0, v = 0.0, up = 1.0;
  for (int i = 1; i <= l; ++i) {
    int d = (int)((n >> (2 * (l - i))) & 3);
    double Ri = ldexp(g.root_size, -i);
    if (d == 0) {
      up = -up;
    } else if (d == 1) {
      v = __dadd_rn(v, up * Ri);
    } else {
      double RH = __dmul_rn(Ri, FMM_H);
      u = (d == 2) ? __dsub_rn(u, RH) : __dadd_rn(u, RH);
      v = __dsub_rn(v, up * (0.5 * Ri));
    }
  }
  return make_double2(__dadd_rn(u, g.root_x), __dadd_rn(v, g.root_y));
}

// adjacentNeighbor by ancestor-sibling-reflect with Table 1; k: 0 L, 1 R, 2 V
__device__ inline int64_t triq_adjacent(int l, int64_t n, int k) {
  // Table 1 packed into constants (no local-memory tables):
  //   D[type][k] = {{2, 3, 1}, {3, 2, 0}, {1, 0, 2}, {0, 1, 3}}     2 bits at 2 (3 type + k)
  //   STAR[type][k] = {{1, 1, 1}, {0, 0, 1}, {0, 1, 0}, {1, 0, 0}}  1 bit at 3 type + k
  constexpr uint32_t DP = 0xd212deu, SP = 0x2a7u;
  if (n < 0) return -1;
  int i = l;  // digit position from the right end
  while (i >= 1) {
    int d = (int)((n >> (2 * (l - i))) & 3);
    if ((SP >> (3 * d + k)) & 1u) break;
    --i;
  }
  if (i < 1) return -1;
  int64_t r = n;
  for (int j = i; j <= l; ++j) {
    int sh = 2 * (l - j);
    int d = (int)((n >> sh) & 3);
    r = (r & ~((int64_t)3 << sh)) | ((int64_t)((DP >> (2 * (3 * d + k))) & 3u) << sh);
  }
  return r;
}

__device__ inline int triq_neighbors(int l, int64_t n, int64_t* out) {
  int64_t Lc = triq_adjacent(l, n, 0), Rc = triq_adjacent(l, n, 1), Vc = triq_adjacent(l, n, 2);
  int64_t VL = triq_adjacent(l, Vc, 0), VR = triq_adjacent(l, Vc, 1);
  int64_t LL = triq_adjacent(l, Lc, 0), RR = triq_adjacent(l, Rc, 1);
  int64_t LV = triq_adjacent(l, Lc, 2), RV = triq_adjacent(l, Rc, 2);
  int64_t VLL = triq_adjacent(l, VL, 0), VRR = triq_adjacent(l, VR, 1), LVR = triq_adjacent(l, LV, 1);
  int64_t all[12] = {Lc, Rc, Vc, VL, VR, LL, RR, LV, RV, VLL, VRR, LVR};
  int c = 0;
  for (int a = 0; a < 12; ++a) {
    if (all[a] < 0 || all[a] == n) continue;
    bool dup = false;
    for (int b = 0; b < c; ++b) dup |= (out[b] == all[a]);
    if (!dup) out[c++] = all[a];
  }
  return c;
}

// ------------------------------------------------------------------ dispatch
__device__ inline bool geo_key(const DGeo& g, double x, double y, uint32_t* key) {
  if (g.tiling == FMM_QUADTREE) return quad_key(g, x, y, key);
  if (g.tiling == FMM_SEPTREE) return sept_key(g, x, y, key);
  return triq_key(g, x, y, key);
}
__device__ inline double2 geo_centre(const DGeo& g, int l, int64_t n) {
  if (g.tiling == FMM_QUADTREE) return quad_centre(g, l, n);
  if (g.tiling == FMM_SEPTREE) return sept_centre(g, l, n);
  return triq_centre(g, l, n);
}
__device__ inline int geo_neighbors(const DGeo& g, int l, int64_t n, int64_t* out) {
  if (l <= 0) return 0;
  if (g.tiling == FMM_QUADTREE) return quad_neighbors(l, n, out);
  if (g.tiling == FMM_SEPTREE) return sept_neighbors(l, n, out);
  return triq_neighbors(l, n, out);
}
