// passes.cu -- FMM evaluation passes on the device (FP64 complex arithmetic):
//   P2M, M2M (upward), L2L + M2L per level (downward), L2P fused with P2P (near field).
// Operators: classical 2D log-kernel forms (PAPER.md P:43 omits them; D10):
//   P2M  Q = sum u_i, a_k = -(1/k) sum u_i (x_i - c)^k
//   M2M  a'_l = -Q z0^l / l + sum_{k=1..l} a_k z0^{l-k} C(l-1, k-1),      z0 = c_child - c_parent
//   M2L  b_l  = w^l (-Q/l + sum_k C(l+k-1, k-1) (-1)^k a_k w^k),  w = 1/(c_M - c_L);
//        b_0  = Q Log(c_L - c_M) + sum_k (-1)^k a_k w^k
//   L2L  b'_l = sum_{k=l..p} b_k C(k, l) w^{k-l},                      w = c_child - c_parent
//   L2P  sum_l b_l (y - c)^l;  P2P  sum_i u_i Log(y - x_i)
#include <stdlib.h>

#include "fmm_internal.cuh"
#include "geometry.cuh"
#include "p2p_math.cuh"

namespace {

constexpr int BS = 2 * FMM_MAX_P + 2;  // binomial table stride

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
// c + a b in four fused multiply-adds (cadd(c, cmul(a, b)) takes two multiplies, two FMAs and two adds)
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cinv(double2 z) {
  double d = 1.0 / (z.x * z.x + z.y * z.y);
  return make_double2(z.x * d, -z.y * d);
}
__device__ __forceinline__ double2 shfl_d2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
// principal Log with canonical +0 imaginary zero (D13)
__device__ __forceinline__ double2 clog_principal(double dx, double dy) {
  dy = __dadd_rn(dy, 0.0);
  return make_double2(0.5 * log(dx * dx + dy * dy), atan2(dy, dx));
}

// ------------------------------------------------------------------ P2M (lane groups per leaf)
// P2M_LPL lanes per leaf (4: 8 leaves per warp; 8 and 16 were slower, 2 slower on the
// clustered C5): each lane accumulates u z^k over every P2M_LPL-th source of its leaf, then
// an xor reduction within the lane group.
#ifndef P2M_LPL
#define P2M_LPL 4
#endif
template <int P>
__global__ void __launch_bounds__(128) k_p2m(const double2* __restrict__ sxy, const double* __restrict__ su,
                                             const int32_t* __restrict__ soff, const double2* __restrict__ cen,
                                             int64_t own_lo, int64_t own_hi, int p, double2* __restrict__ mp) {
  // leaves [own_lo, own_hi): every leaf on one rank; on a multi-rank tree this rank's own source
  // leaves only (the halo leaves it keeps for P2P belong to other ranks' partial trees, and the
  // rest of the multipole tree was zeroed)
  const int64_t leaf = own_lo + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / P2M_LPL;
  const int sub = threadIdx.x & (P2M_LPL - 1);
  const bool lvalid = leaf < own_hi;
  const int s0 = lvalid ? soff[leaf] : 0, s1 = lvalid ? soff[leaf + 1] : 0;
  const double2 c = lvalid ? cen[leaf] : make_double2(0.0, 0.0);
  double Sr[P + 1], Si[P + 1];
#pragma unroll
  for (int k = 0; k <= P; ++k) Sr[k] = Si[k] = 0.0;
  // the next source of the lane is loaded before the current one's power chain (software
  // pipelining: the load latency overlaps the chain)
  double2 x = s0 + sub < s1 ? sxy[s0 + sub] : c;
  double u = s0 + sub < s1 ? su[s0 + sub] : 0.0;
  for (int i = s0 + sub; i < s1; i += P2M_LPL) {
    const bool more = i + P2M_LPL < s1;
    const double2 xn = more ? sxy[i + P2M_LPL] : c;
    const double un = more ? su[i + P2M_LPL] : 0.0;
    double zr = x.x - c.x, zi = x.y - c.y;
    double pr = u, pi = 0.0;  // u z^k
    Sr[0] += u;
#pragma unroll
    for (int k = 1; k <= P; ++k) {
      double nr = pr * zr - pi * zi, ni = pr * zi + pi * zr;
      pr = nr;
      pi = ni;
      Sr[k] += pr;
      Si[k] += pi;
    }
    x = xn;
    u = un;
  }
#pragma unroll
  for (int k = 0; k <= P; ++k) {
#pragma unroll
    for (int o = 1; o < P2M_LPL; o <<= 1) {
      Sr[k] += __shfl_xor_sync(0xffffffffu, Sr[k], o);
      Si[k] += __shfl_xor_sync(0xffffffffu, Si[k], o);
    }
  }
  if (!lvalid) return;
  double2* out = mp + leaf * (p + 1);
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    if (k <= p && sub == (k & (P2M_LPL - 1))) {
      out[k] = (k == 0) ? make_double2(Sr[0], 0.0) : make_double2(-Sr[k] / k, -Si[k] / k);
    }
  }
}

// ------------------------------------------------------------------ M2M (one warp per parent, lane = coefficient)
// All B children's multipoles are staged in shared memory first, with one load latency for all
// of them, and lane k then runs the B children's Horner chains in step (B independent chains:
// the latency of one is hidden by the others); the children are added in ascending order as
// before.  The binomials C(k - 1, j - 1) of lane k's row are read from the global table (L1)
// in the chain: staging a 32 x 32 table per block of four parents cost more than it saved.
template <int B>
__global__ void __launch_bounds__(128) k_m2m(int64_t par0, int64_t nparents, int64_t span_l,
                                             const int32_t* __restrict__ soff,
                                             const double2* __restrict__ cen_par, const double2* __restrict__ cen_ch,
                                             const double2* __restrict__ mp_ch, int p, const double* __restrict__ binom,
                                             double2* __restrict__ mp_par) {
  __shared__ double2 s_a[4][B][32];
  __shared__ double2 s_z[4][B];   // c_child - c_parent of the staged children
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t P = par0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);  // parents [par0, nparents)
  if (P >= nparents) return;
  const double2 cp = cen_par[P];
  const int k = lane;  // p <= 31: one coefficient per lane
  // non-empty children, in ascending order, staged at the front of s_a (empty children add
  // nothing: clustered trees have many)
  int nc = 0;
#pragma unroll
  for (int ch = 0; ch < B; ++ch) {
    const int64_t c = P * B + ch;
    if (soff[(c + 1) * span_l] == soff[c * span_l]) continue;
    s_a[w][nc][lane] = lane <= p ? mp_ch[c * (p + 1) + lane] : make_double2(0.0, 0.0);
    if (lane == 0) {
      const double2 cc = cen_ch[c];
      s_z[w][nc] = make_double2(cc.x - cp.x, cc.y - cp.y);
    }
    ++nc;
  }
  __syncwarp();
  double2 acc = make_double2(0.0, 0.0);
  if (k == 0) {
    for (int q = 0; q < nc; ++q) acc.x += s_a[w][q][0].x;
  } else if (k <= p) {
    // up to 4 children's Horner chains in step (independent: their latencies overlap)
    for (int q0 = 0; q0 < nc; q0 += 4) {
      double2 h[4], z0[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool v = q0 + q < nc;
        h[q] = make_double2(v ? -s_a[w][q0 + q][0].x / k : 0.0, 0.0);
        z0[q] = v ? s_z[w][q0 + q] : make_double2(0.0, 0.0);
      }
      const double* crow = binom + (k - 1) * BS - 1;  // crow[j] = C(k - 1, j - 1)
      for (int j = 1; j <= k; ++j) {
        const double cj = __ldg(crow + j);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 a = q0 + q < nc ? s_a[w][q0 + q][j] : make_double2(0.0, 0.0);
          h[q] = cadd(cmul(h[q], z0[q]), cscale(cj, a));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q0 + q < nc) acc = cadd(acc, h[q]);
    }
  }
  if (k <= p) mp_par[P * (p + 1) + k] = acc;
}

// ------------------------------------------------------------------ downward v2 (templated on P >= p)
// One warp per target cell t with targets; lane l owns local coefficient b_l.
//  * L2L from the parent (l >= 2): Horner in w = c_t - c_par over k = p..l.
//  * M2L over E4(t) in batches of 16 sources.  Phase A (lane j = source j): w_j = 1/(c_s - c_t),
//    all powers w_j^k -> shared memory, Log(c_t - c_s) (D13 iii) and Q_j.  Phase B, per source:
//    lane l forms a~_l = (-1)^l a_l w^l (Pascal-scaled form), then
//    b_l += w^l (sum_k C(l+k-1, k-1) a~_k - Q/l) with its binomial row C(l+k-1, k-1) held in
//    registers; lane 0 adds Q Log(c_t - c_s) + sum_k a~_k.
template <int P>
__global__ void __launch_bounds__(128) k_down2(int l, int B, int64_t cell0, int64_t ncells, int64_t span_l,
                                               const int32_t* __restrict__ toff, int64_t leaf_lo, int64_t leaf_hi,
                                               const double2* __restrict__ cen_l, const double2* __restrict__ cen_par,
                                               const double2* __restrict__ loc_par, const int32_t* __restrict__ cand,
                                               const unsigned long long* __restrict__ e4mask,
                                               const double2* __restrict__ mp_l, int p,
                                               const double* __restrict__ binom, double2* __restrict__ loc_l) {
  constexpr int NB = 16;  // sources per batch
  __shared__ double2 s_pw[4][NB][P + 1];
  __shared__ double2 s_lg[4][NB];
  __shared__ double s_q[4][NB];
  __shared__ double2 s_at[4][32];
  const int64_t t = cell0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 3;
  if (t >= ncells) return;
  const int64_t tlo = max(t * span_l, leaf_lo), thi = min((t + 1) * span_l, leaf_hi);
  if (thi <= tlo || toff[thi] == toff[tlo]) return;  // no targets of this rank below t
  const double2 ct = cen_l[t];
  double2 acc = make_double2(0.0, 0.0);
  const bool out_lane = lane <= p;
  // binomial row of this lane: C(l+k-1, k-1), k = 1..P (0 beyond p)
  double cb[P];
#pragma unroll
  for (int k = 1; k <= P; ++k) cb[k - 1] = (k <= p && out_lane) ? binom[(lane + k - 1) * BS + (k - 1)] : 0.0;
  const double inv_l = lane > 0 ? 1.0 / lane : 0.0;
  const int64_t par = t / B;
  if (l >= 2) {
    const double2 cpp = cen_par[par];
    const double2 wv = make_double2(ct.x - cpp.x, ct.y - cpp.y);
    const double2* bp = loc_par + par * (p + 1);
    for (int k = p; k >= 0; --k) {
      const double2 bk = bp[k];
      if (k >= lane && out_lane) acc = cadd(cmul(acc, wv), cscale(binom[k * BS + lane], bk));
    }
  }
  unsigned long long mask = e4mask[t];
  const int32_t* cd = cand + par * FMM_CAND_MAX;
  while (mask) {
    // ---- phase A: up to NB sources, lane j handles source j
    int nb = 0;
    int src_j = -1;
    {
      unsigned long long mm = mask;
      for (int j = 0; j < NB && mm; ++j) {
        int i = __ffsll((long long)mm) - 1;
        mm &= mm - 1;
        if (lane == j) src_j = cd[i];
        ++nb;
      }
      mask = mm;
    }
    if (lane < nb) {
      const double2 cs = cen_l[src_j];
      const double zx = cs.x - ct.x, zy = cs.y - ct.y;
      const double d = 1.0 / (zx * zx + zy * zy);
      const double2 wv = make_double2(zx * d, -zy * d);
      double2 pw = make_double2(1.0, 0.0);
      s_pw[w][lane][0] = pw;
#pragma unroll
      for (int k = 1; k <= P; ++k) {
        pw = cmul(pw, wv);
        s_pw[w][lane][k] = pw;
      }
      s_lg[w][lane] = clog_principal(ct.x - cs.x, ct.y - cs.y);  // Log(c_L - c_M), D13 (iii)
      s_q[w][lane] = mp_l[(int64_t)src_j * (p + 1)].x;
    }
    __syncwarp();
    // ---- phase B
    for (int j = 0; j < nb; ++j) {
      const int s = __shfl_sync(0xffffffffu, src_j, j);
      const double2 a = out_lane ? mp_l[(int64_t)s * (p + 1) + lane] : make_double2(0.0, 0.0);
      const double2 pwl = lane <= P ? s_pw[w][j][min(lane, P)] : make_double2(0.0, 0.0);
      double2 at = cmul(a, pwl);
      if (lane & 1) at = make_double2(-at.x, -at.y);
      s_at[w][lane] = at;
      __syncwarp();
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int k = 1; k <= (P < 32 ? P : 31); ++k) {  // p <= 31: coefficient 32 never exists
        const double2 ak = s_at[w][k];
        sr = fma(cb[k - 1], ak.x, sr);
        si = fma(cb[k - 1], ak.y, si);
      }
      const double Q = s_q[w][j];
      if (lane == 0) {
        const double2 lg = s_lg[w][j];
        acc.x += Q * lg.x + sr;
        acc.y += Q * lg.y + si;
      } else if (out_lane) {
        acc = cadd(acc, cmul(pwl, make_double2(fma(-Q, inv_l, sr), si)));
      }
      __syncwarp();
    }
  }
  if (out_lane) loc_l[t * (p + 1) + lane] = acc;
}

template <int P>
void launch_p2m(fmm_tree_s* t) {
  const Geo& G = t->g;
  const int64_t nl = t->leaf_hi - t->leaf_lo;
  if (nl <= 0) return;
  k_p2m<P><<<(unsigned)((nl * P2M_LPL + 127) / 128), 128, 0, t->stream>>>(
      t->sxy, t->su, t->soff, t->centre + G.lvl_off[G.L], t->leaf_lo, t->leaf_hi, G.p,
      t->mp + G.lvl_off[G.L] * (G.p + 1));
}

}  // namespace

// cells [c0, c1) of level l that hold a leaf of this rank's range (every cell on one rank)
static void level_range(const fmm_tree_s* t, int l, int64_t* c0, int64_t* c1) {
  const Geo& G = t->g;
  const int64_t span = G.ncells[G.L - l];  // B^(L-l)
  if (t->leaf_hi <= t->leaf_lo) {
    *c0 = *c1 = 0;
    return;
  }
  *c0 = t->leaf_lo / span;
  *c1 = (t->leaf_hi + span - 1) / span;
}

int fmm_stage_upward(fmm_tree_s* t) {
  const Geo& G = t->g;
  cudaStream_t s = t->stream;
  int p = G.p;
  // multi-rank: the partial multipole tree is zero outside this rank's own cells (the all-reduce
  // sums every rank's tree); P2M / M2M then run over the rank's cells only
  if (t->cfg.nranks > 1)
    FMM_CUDA_TRY(cudaMemsetAsync(t->mp, 0, sizeof(double2) * (size_t)G.total_cells * (p + 1), s));
  if (p <= 8) launch_p2m<8>(t);
  else if (p <= 12) launch_p2m<12>(t);
  else if (p <= 16) launch_p2m<16>(t);
  else if (p <= 20) launch_p2m<20>(t);
  else if (p <= 24) launch_p2m<24>(t);
  else if (p <= 28) launch_p2m<28>(t);
  else launch_p2m<32>(t);
  t->launches++;
  for (int l = G.L - 1; l >= 1; --l) {
    int64_t c0, c1;
    level_range(t, l, &c0, &c1);
    if (c1 <= c0) continue;
    auto m2m = G.B == 7 ? k_m2m<7> : k_m2m<4>;
    m2m<<<(unsigned)(((c1 - c0) * 32 + 127) / 128), 128, 0, s>>>(
        c0, c1, G.ncells[G.L - l - 1] /* B^(L-l-1) */, t->soff, t->centre + G.lvl_off[l],
        t->centre + G.lvl_off[l + 1], t->mp + G.lvl_off[l + 1] * (p + 1), p, t->binom, t->mp + G.lvl_off[l] * (p + 1));
    t->launches++;
  }
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

// ------------------------------------------------------------------ downward with FP64 tensor cores
// M2L in the Pascal-scaled form: for a batch of NB sources s of E4(t),
//   Y[l][s] = sum_{k=1..p} C(l+k-1, k-1) a~_{s,k},   a~_{s,k} = (-1)^k a_{s,k} w_s^k,
//   b_l += w_s^l (Y[l][s] - Q_s / l)   (l >= 1),     b_0 += Q_s Log(c_t - c_s) + Y[0][s]
// The contraction Y = Cb * A~ over the rows l = 1..p (Cb: p x p real, stored as
// (-1)^k C(l+k-1, k-1) so that the staged A~ is a_{s,k} w_s^k without the sign; A~: p x 2 NB, real
// and imaginary parts as columns) runs on DMMA (mma.sync m8n8k4 f64, IEEE FP64 multiply-adds): Cb
// lives in the A fragments of the warp's registers, A~ is staged in shared memory.  Row l = 0 has
// C(k-1, k-1) = 1: Y[0][s] is the plain sum of the a~_{s,k}; when P is a multiple of 8 the staging
// lanes form it (ROW0) and the row tiles cover l = 1..P, so that p = 24 (16) needs 3 (2) row tiles
// of 8 instead of 4 (3); otherwise row 0 rides in the first tile for free.  b_0's Q_s Log(c_t - c_s)
// terms are formed before the batch loop with one source per lane (inside the loop only the 8
// lanes j = 0 would run the ~70-instruction Log, once per batch).  Fragment layouts
// (m8n8k4 .f64): A[r][c] at lane 4r + c; B[k][n] at lane 4n + k; C[r][2c + {0,1}] at lane 4r + c.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// shared memory of one k_down_mma block (dynamic): the binomial A fragments and the 1/r table
// (copied from the tree's precomputed fmm_down_afr_fill image), then per warp: powers, a~, L2L
// part, Q, source ids.  b_0's Log reads the P2P log / atan tables from global memory (L1).
template <int P>
struct DownSmem {
  static constexpr bool ROW0 = P % 8 == 0;  // row l = 0 formed outside the DMMA tiles
  static constexpr int R0 = ROW0 ? 1 : 0;   // first row of the tiles
  static constexpr int NB = 8, MT = ROW0 ? P / 8 : (P + 8) / 8, KT = P / 4;  // rows R0 .. R0 + 8 MT - 1
  static constexpr int afr_n = MT * KT * 32 + 8 * MT + 8;  // A fragments + 1/r table, r = 0..8 MT (+ padding)
  static constexpr size_t afr = sizeof(double) * afr_n;
  // a~ is stored as separate real and imaginary rows of PS doubles per source (the B fragment of a
  // lane is one double); PS = 4 or 12 mod 16 keeps the 8 rows a fragment load touches on distinct banks
  static constexpr int PS = (P % 16 == 4 || P % 16 == 12) ? P : P + 4;
  static constexpr size_t warp = sizeof(double2) * (NB * (P + 1) + NB * PS + 32) + sizeof(double) * NB +
                                 sizeof(int) * FMM_CAND_MAX;
  static constexpr size_t bytes = afr + 4 * warp;
};

#ifndef DOWN_MINB
// resident blocks per SM (register budget 128 / 102 / 85): measured with the 33 KB blocks of the
// precomputed fragment image -- p = 24 at 5 blocks (96 registers, 12 bytes of spill) is 3-4 %
// faster than at 4, p <= 20 at 6 blocks (80 registers) 2.5-3.5 % faster than at 5; p >= 28 spills at 5
#define DOWN_MINB(P) ((P) >= 28 ? 4 : ((P) >= 24 ? 5 : 6))
#endif
template <int P>
__global__ void __launch_bounds__(128, DOWN_MINB(P)) k_down_mma(int l, int B, int64_t cell0, int64_t ncells,
                                                     int64_t span_l,
                                                     const int32_t* __restrict__ toff, int64_t leaf_lo,
                                                     int64_t leaf_hi, const double2* __restrict__ cen_l,
                                                     const double2* __restrict__ cen_par,
                                                     const double2* __restrict__ loc_par,
                                                     const int32_t* __restrict__ cand,
                                                     const unsigned long long* __restrict__ e4mask,
                                                     const double2* __restrict__ mp_l, int p,
                                                     const double* __restrict__ binom, const double* __restrict__ tabs,
                                                     const double* __restrict__ afr, double2* __restrict__ loc_l) {
  using S = DownSmem<P>;
  constexpr int NB = S::NB, MT = S::MT, KT = S::KT, R0 = S::R0, PS = S::PS;
  constexpr bool ROW0 = S::ROW0;
  extern __shared__ double2 dsm[];
  double* s_afr = (double*)dsm;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  char* wb = (char*)dsm + S::afr + w * S::warp;
  double2* s_pw = (double2*)wb;          // [NB][P+1] w_s^k
  double* s_at = (double*)(s_pw + NB * (P + 1));  // [NB][2][PS] Re / Im rows of a~_{s,k}, k = 1..P
  double2* s_b = (double2*)(s_at + 2 * NB * PS);  // [32]      L2L part
  double* s_q = (double*)(s_b + 32);     // [NB]
  int* s_src = (int*)(s_q + NB);         // [FMM_CAND_MAX] E4(t)
  // the cell's own loads (everything that depends on t alone: target counts, E4 mask, centres, the
  // parent's candidates and local expansion), issued before the block's fragment copy so that one
  // memory round trip covers them all; a warp past the last cell reads the last cell's
  const int64_t t = cell0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);  // cells [cell0, ncells)
  const int64_t tc = min(t, ncells - 1), par = tc / B;
  const int64_t tlo = max(tc * span_l, leaf_lo), thi = min((tc + 1) * span_l, leaf_hi);
  const int n_lo = toff[tlo], n_hi = toff[thi];
  const unsigned long long mask = e4mask[tc];
  const double2 ct = cen_l[tc];
  const int32_t* cd = cand + par * FMM_CAND_MAX;
  const int cd0 = cd[lane], cd1 = cd[lane + 32];
  double2 cpp = make_double2(0.0, 0.0), lpar = make_double2(0.0, 0.0);
  if (l >= 2) {
    cpp = cen_par[par];
    if (lane <= p) lpar = loc_par[par * (p + 1) + lane];
  }
  // A fragments Cb[r][k] = (-1)^k C(r+k-1, k-1) (the sign of a~ folded in; row r = 8 mt + ln/4 + R0,
  // column k = 4 kt + ln%4 + 1, at (mt KT + kt) 32 + ln) and the 1/r table behind them: one
  // coalesced copy of the image fmm_down_afr_fill built for this order
  for (int i = threadIdx.x; i < S::afr_n; i += blockDim.x) s_afr[i] = afr[i];
  const double* s_invr = s_afr + MT * KT * 32;  // [8 MT + 1] 1/r (0 for r = 0)
  __syncthreads();
  // b_0's Log: the compact log / atan tables of the P2P math, read from global memory
  const double2* a_log = (const double2*)tabs + P2P_TAB_LOGC / 2;
  const double2* a_atan = (const double2*)tabs + P2P_TAB_ATANC / 2;
  if (t >= ncells) return;
  if (thi <= tlo || n_hi == n_lo) return;  // no targets of this rank below t
  // ---- E4(t) source ids, ascending: lane i places candidates i and i + 32 by prefix popcount
  {
    const unsigned lo = (unsigned)mask, hi = (unsigned)(mask >> 32), below = (1u << lane) - 1u;
    if ((lo >> lane) & 1u) s_src[__popc(lo & below)] = cd0;
    if ((hi >> lane) & 1u) s_src[__popc(lo) + __popc(hi & below)] = cd1;
  }
  const int nsrc = __popcll(mask);
  // ---- L2L (lane = coefficient): Horner in w = c_t - c_par over k = p..l
  {
    double2 acc = make_double2(0.0, 0.0);
    if (l >= 2) {
      const double2 wv = make_double2(ct.x - cpp.x, ct.y - cpp.y);
      s_b[lane] = lpar;
      __syncwarp();
#pragma unroll
      for (int k = P; k >= 0; --k) {  // unrolled: the binomial loads leave the Horner chain
        if (k > p) continue;
        const double2 bk = s_b[k];
        if (k >= lane && lane <= p) acc = cfma(acc, wv, cscale(binom[k * BS + lane], bk));
      }
      __syncwarp();
    }
    s_b[lane] = acc;
  }
  double2 acc[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) acc[mt] = make_double2(0.0, 0.0);
  __syncwarp();
  // ---- b_0 of the M2L, partial per lane: Q_s Log(c_t - c_s) (D13 iii; canonical +0 imaginary zero;
  // table-driven), one source per lane; ROW0 adds the Y[0][s] of the staging lanes j = 0 below
  double2 b0 = make_double2(0.0, 0.0);
  for (int i = lane; i < nsrc; i += 32) {
    const int src = s_src[i];
    const double2 cs = cen_l[src];
    const double Q = mp_l[(int64_t)src * (p + 1)].x;
    const double dx = ct.x - cs.x, dy = __dadd_rn(ct.y - cs.y, 0.0);
    b0.x = fma(Q, 0.5 * p2p_log<P2P_LOGC_N, const double2*>(fma(dx, dx, dy * dy), a_log), b0.x);
    b0.y = fma(Q, p2p_atan2<false, const double2*>(dy, dx, a_atan), b0.y);
  }
  for (int b0s = 0; b0s < nsrc; b0s += NB) {
    const int nb = min(NB, nsrc - b0s);
    // lane = (source s = lane / 4, residue j = lane % 4) owns exponents k = 4m + j: it loads
    // a_{s,k} (all its loads first), forms w^k and a_{s,k} w^k (the (-1)^k of a~ is in Cb) and
    // (ROW0) its share of Y[0][s] = sum_k (-1)^k a_{s,k} w^k ((-1)^k = (-1)^j)
    {
      constexpr int NM = P / 4 + 1;
      const int s = lane >> 2, j = lane & 3;
      double2 y0 = make_double2(0.0, 0.0);
      if (s < nb) {
        const int src = s_src[b0s + s];
        const double2* ab = mp_l + (int64_t)src * (p + 1);
        double2 av[NM];
#pragma unroll
        for (int m = 0; m < NM; ++m) av[m] = (4 * m + j <= p) ? ab[4 * m + j] : make_double2(0.0, 0.0);
        const double2 cs = cen_l[src];
        const double zx = cs.x - ct.x, zy = cs.y - ct.y;
        const double d = p2p_rcp(fma(zx, zx, zy * zy));
        const double2 wv = make_double2(zx * d, -zy * d);
        const double2 w2 = cmul(wv, wv);
        const double2 w4 = cmul(w2, w2);
        double2 pw = j == 0 ? make_double2(1.0, 0.0) : (j == 1 ? wv : (j == 2 ? w2 : cmul(w2, wv)));
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          const int k = 4 * m + j;
          if (k <= P) s_pw[s * (P + 1) + k] = pw;
          if (k >= 1 && k <= P) {
            const double2 at = cmul(av[m], pw);  // (-1)^k is in Cb
            s_at[(2 * s) * PS + k - 1] = at.x;
            s_at[(2 * s + 1) * PS + k - 1] = at.y;
            if (ROW0) y0 = cadd(y0, at);
          }
          pw = cmul(pw, w4);
        }
        if (j == 0) s_q[s] = av[0].x;
      }
      if (ROW0) {  // every lane's share, signed (lanes past nb carry 0): the final sum over lanes adds them
        if (j & 1) {
          b0.x -= y0.x;
          b0.y -= y0.y;
        } else {
          b0.x += y0.x;
          b0.y += y0.y;
        }
      }
    }
    __syncwarp();
    {
      // both column tiles (sources 0-3 and 4-7 of the batch) in one sweep over k: each A fragment
      // is read from shared memory once for the two DMMAs
      const bool two = nb > 4;
      double d[2][MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) d[0][mt][0] = d[0][mt][1] = d[1][mt][0] = d[1][mt][1] = 0.0;
      const int bs = lane >> 3, bc = (lane >> 2) & 1;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const double b0f = s_at[(2 * bs + bc) * PS + 4 * kt + (lane & 3)];
        const double b1f = two ? s_at[(2 * (4 + bs) + bc) * PS + 4 * kt + (lane & 3)] : 0.0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = s_afr[(mt * KT + kt) * 32 + lane];
          dmma884(d[0][mt][0], d[0][mt][1], a, b0f);
          if (two) dmma884(d[1][mt][0], d[1][mt][1], a, b1f);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int s = 4 * nt + (lane & 3);
        if (s < nb) {
          const double Q = s_q[s];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int r = 8 * mt + (lane >> 2) + R0;
            if (r > P) continue;
            if (!ROW0 && r == 0) {
              acc[mt].x += d[nt][mt][0];
              acc[mt].y += d[nt][mt][1];
            } else {
              const double2 pw = s_pw[s * (P + 1) + r];
              acc[mt] = cfma(pw, make_double2(fma(-Q, s_invr[r], d[nt][mt][0]), d[nt][mt][1]), acc[mt]);
            }
          }
        }
      }
    }
    __syncwarp();
  }
  // sum the 4 lanes (lane % 4) that hold the same row, then write b_l (+ L2L part)
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    acc[mt].x += __shfl_xor_sync(0xffffffffu, acc[mt].x, 1);
    acc[mt].y += __shfl_xor_sync(0xffffffffu, acc[mt].y, 1);
    acc[mt].x += __shfl_xor_sync(0xffffffffu, acc[mt].x, 2);
    acc[mt].y += __shfl_xor_sync(0xffffffffu, acc[mt].y, 2);
    const int r = 8 * mt + (lane >> 2) + R0;
    if (!ROW0 && r == 0) continue;  // written with b0 below
    if ((lane & 3) == 0 && r <= p) loc_l[t * (p + 1) + r] = cadd(acc[mt], s_b[r]);
  }
  // b_0: the lanes' partials (butterfly: a fixed order), plus row 0 of the first tile when it rides there
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    b0.x += __shfl_xor_sync(0xffffffffu, b0.x, o);
    b0.y += __shfl_xor_sync(0xffffffffu, b0.y, o);
  }
  if (lane == 0) {
    if (!ROW0) b0 = cadd(b0, acc[0]);
    loc_l[t * (p + 1)] = cadd(b0, s_b[0]);
  }
}

int fmm_down_order(int p) { return p <= 8 ? 8 : (p + 3) / 4 * 4; }

template <int P>
static int afr_fill(const double* binom, double* out) {
  using S = DownSmem<P>;
  for (int i = 0; i < S::MT * S::KT * 32; ++i) {
    const int ln = i & 31, kt = (i >> 5) % S::KT, mt = (i >> 5) / S::KT;
    const int r = 8 * mt + (ln >> 2) + S::R0, k = 4 * kt + (ln & 3) + 1;
    // rows r > p are never written and columns k > p meet zero coefficients, so the image
    // depends on the order P only
    const double c = binom[(size_t)(r + k - 1) * BS + (k - 1)];
    out[i] = (k & 1) ? -c : c;
  }
  double* invr = out + S::MT * S::KT * 32;
  for (int i = 0; i <= 8 * S::MT; ++i) invr[i] = i > 0 ? 1.0 / i : 0.0;
  return S::afr_n;
}

int fmm_down_afr_fill(int P, const double* binom, double* out) {
  switch (P) {
    case 8: return afr_fill<8>(binom, out);
    case 12: return afr_fill<12>(binom, out);
    case 16: return afr_fill<16>(binom, out);
    case 20: return afr_fill<20>(binom, out);
    case 24: return afr_fill<24>(binom, out);
    case 28: return afr_fill<28>(binom, out);
    default: return afr_fill<32>(binom, out);
  }
}

template <int P>
static void launch_down(fmm_tree_s* t, int l) {
  const Geo& G = t->g;
  const int p = G.p;
  int64_t c0, c1;
  level_range(t, l, &c0, &c1);
  if (c1 <= c0) return;
  const int64_t nc = c1 - c0;
  static const bool simt = getenv("FMM_M2L_SIMT") && getenv("FMM_M2L_SIMT")[0] == '1';
  if (!simt) {
    // per device (a process may drive several GPUs); a failure surfaces as the launch error
    cudaFuncSetAttribute(k_down_mma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DownSmem<P>::bytes);
    k_down_mma<P><<<(unsigned)((nc * 32 + 127) / 128), 128, DownSmem<P>::bytes, t->stream>>>(
        l, G.B, c0, c1, G.ncells[G.L - l] /* B^(L-l) */, t->toff, t->leaf_lo, t->leaf_hi, t->centre + G.lvl_off[l],
        t->centre + G.lvl_off[l - 1], t->loc + G.lvl_off[l - 1] * (p + 1), t->cand + G.lvl_off[l - 1] * FMM_CAND_MAX,
        t->e4mask + G.lvl_off[l], t->mp + G.lvl_off[l] * (p + 1), p, t->binom, t->p2p_tab, t->afr,
        t->loc + G.lvl_off[l] * (p + 1));
    return;
  }
  k_down2<P><<<(unsigned)((nc * 32 + 127) / 128), 128, 0, t->stream>>>(
      l, G.B, c0, c1, G.ncells[G.L - l] /* B^(L-l) */, t->toff, t->leaf_lo, t->leaf_hi, t->centre + G.lvl_off[l],
      t->centre + G.lvl_off[l - 1], t->loc + G.lvl_off[l - 1] * (p + 1), t->cand + G.lvl_off[l - 1] * FMM_CAND_MAX,
      t->e4mask + G.lvl_off[l], t->mp + G.lvl_off[l] * (p + 1), p, t->binom, t->loc + G.lvl_off[l] * (p + 1));
}

// m2l_dense.cu (NEXT-3): per-offset operators on DMMA, quadtree, FMM_M2L_DENSE=1
bool fmm_m2l_dense_enabled(const fmm_tree_s* t);
int fmm_m2l_dense_lmin(int L);
int fmm_m2l_dense_level(fmm_tree_s* t, int l, int64_t c0, int64_t c1, double* Tfrag);
size_t fmm_m2l_dense_table_bytes(int p);

int fmm_stage_downward(fmm_tree_s* t) {
  const Geo& G = t->g;
  const int p = G.p;
  double* Tfrag = nullptr;
  const int ldense = fmm_m2l_dense_enabled(t) ? fmm_m2l_dense_lmin(G.L) : G.L + 1;
  if (ldense <= G.L) FMM_CUDA_TRY(cudaMallocAsync((void**)&Tfrag, fmm_m2l_dense_table_bytes(p), t->stream));
  for (int l = 1; l <= G.L; ++l) {
    if (l >= ldense) {
      int64_t c0, c1;
      level_range(t, l, &c0, &c1);
      if (c1 > c0) {
        int e = fmm_m2l_dense_level(t, l, c0, c1, Tfrag);
        if (e) return e;
      }
      continue;
    }
    if (p <= 8) launch_down<8>(t, l);
    else if (p <= 12) launch_down<12>(t, l);
    else if (p <= 16) launch_down<16>(t, l);
    else if (p <= 20) launch_down<20>(t, l);
    else if (p <= 24) launch_down<24>(t, l);
    else if (p <= 28) launch_down<28>(t, l);
    else launch_down<32>(t, l);
    t->launches++;
  }
  if (Tfrag) cudaFreeAsync(Tfrag, t->stream);
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

