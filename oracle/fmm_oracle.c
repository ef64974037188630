/*
 * fmm_oracle.c -- plain, slow, obviously-correct CPU ORACLE of the hierarchical
 * 2D FMM of arXiv:1204.3105 (square quadtree, septree, triangle-quadtree).
 *
 * TEST INFRASTRUCTURE ONLY (see fmm_oracle.h).  Shares no code with the CUDA
 * product path.  Written from the paper, step by step in its order and notation:
 *   P:n  = /root/reference/PAPER.md line n;  D<k> = DESIGN.md reading k.
 *
 * Arithmetic is IEEE binary64; build with -O2 -ffp-contract=off (no FMA
 * contraction) so that keys and centres follow the exact expression sequences
 * stated in D11/D12.  OpenMP parallel loops only distribute independent cells /
 * targets; per-target and per-cell summation orders are fixed, so results do
 * not depend on the thread count.
 */
#include "fmm_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define MAXD 48 /* max GBT digits handled (addresses have <= L+2 digits) */

static const double S3 = 1.7320508075688772; /* sqrt(3) rounded to binary64 (D11) */
static const double H = 0.8660254037844386;  /* sqrt(3)/2 rounded to binary64 (D11) */

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* thread count of the OpenMP loops (bench.py times the oracle at 1 thread and at all cores;
 * results are identical at any count) */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

static int branching(int tiling) { return tiling == ORC_SEPT ? 7 : 4; }

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

/* digit t_i (1-based, MSB first) of an l-digit base-B address n */
static int digit_at(int64_t n, int B, int l, int i) { return (int)((n / ipow(B, l - i)) % B); }

/* ======================================================================
 * 1. GBT arithmetic  (table of Fig. 4(b))
 * ====================================================================== */

/* Fig. 4(b): pairwise sums of unit digits, printed as base-7
 * numerals (e.g. 63 = carry 6, digit 3).  Row/column 0 is the identity (D4). */
static const int GBT_TABLE[7][7] = {
    {0, 1, 2, 3, 4, 5, 6},     {1, 63, 15, 2, 0, 6, 64}, {2, 15, 14, 26, 3, 0, 1},
    {3, 2, 26, 25, 31, 4, 0},  {4, 0, 3, 31, 36, 42, 5}, {5, 6, 0, 4, 42, 41, 53},
    {6, 64, 1, 0, 5, 53, 52},
};

/* Add a single digit d at position pos of an LSB-first digit array, carrying the
 * high digit of every two-digit table result into the next position (D4). */
static void gbt_add_digit_at(int32_t* dig, int32_t* len, int pos, int d) {
  while (d != 0) {
    if (pos >= MAXD) abort();
    if (pos >= *len) {
      for (int k = *len; k <= pos; ++k) dig[k] = 0;
      *len = pos + 1;
    }
    int s = GBT_TABLE[dig[pos]][d];
    dig[pos] = s % 10;
    d = s / 10;
    ++pos;
  }
}

static int gbt_trim(const int32_t* dig, int len) {
  while (len > 1 && dig[len - 1] == 0) --len;
  return len;
}

int orc_gbt_add(const int32_t* a, int32_t la, const int32_t* b, int32_t lb, int32_t* out) {
  int32_t tmp[MAXD];
  int32_t len = la;
  for (int i = 0; i < la; ++i) tmp[i] = a[i];
  for (int i = 0; i < lb; ++i) gbt_add_digit_at(tmp, &len, i, b[i]);
  len = gbt_trim(tmp, len);
  for (int i = 0; i < len; ++i) out[i] = tmp[i];
  return len;
}

/* opposite unit direction, digit-wise: 1<->4, 2<->5, 3<->6 (D5) */
int orc_gbt_negate(const int32_t* a, int32_t la, int32_t* out) {
  static const int NEG[7] = {0, 4, 5, 6, 1, 2, 3};
  for (int i = 0; i < la; ++i) out[i] = NEG[a[i]];
  return la;
}

/* t0^m by the zero-extension relation of P:168:
 *   j0^m = j0^{m-1} (*) [1+(j mod 6)]0^{m-1} (*) [1+(j mod 6)]0^{m-1}            */
int orc_gbt_zero_extend(int32_t j, int32_t m, int32_t* out) {
  if (m == 0) {
    out[0] = j;
    return 1;
  }
  int32_t a[MAXD], b[MAXD], t[MAXD];
  int la = orc_gbt_zero_extend(j, m - 1, a);
  int lb = orc_gbt_zero_extend(1 + (j % 6), m - 1, b);
  int lt = orc_gbt_add(a, la, b, lb, t);
  return orc_gbt_add(t, lt, b, lb, out);
}

static int index_to_digits7(int64_t n, int32_t* d) {
  int len = 0;
  do {
    d[len++] = (int32_t)(n % 7);
    n /= 7;
  } while (n > 0);
  return len;
}

static int64_t digits7_to_index(const int32_t* d, int len) {
  int64_t n = 0;
  for (int i = len - 1; i >= 0; --i) n = n * 7 + d[i];
  return n;
}

int orc_gbt_index_add(int64_t a, int64_t b, int64_t* out) {
  int32_t da[MAXD], db[MAXD], dr[MAXD];
  int la = index_to_digits7(a, da), lb = index_to_digits7(b, db);
  int lr = orc_gbt_add(da, la, db, lb, dr);
  if (lr > 21) return ORC_EDOMAIN;
  *out = digits7_to_index(dr, lr);
  return ORC_OK;
}

/* ======================================================================
 * 2. Tilings: Children / Parent / Neighbors / NeighborsE4
 * ====================================================================== */

int64_t orc_num_cells(const orc_config* c, int32_t level) { return ipow(branching(c->tiling), level); }

/* --- quadtree: Morton Z order, child digit = 2*ybit + xbit (D7) --- */
static int64_t morton_encode(int64_t i, int64_t j, int l) {
  int64_t k = 0;
  for (int b = 0; b < l; ++b) k |= (((i >> b) & 1) << (2 * b)) | (((j >> b) & 1) << (2 * b + 1));
  return k;
}
static void morton_decode(int64_t k, int l, int64_t* i, int64_t* j) {
  *i = 0;
  *j = 0;
  for (int b = 0; b < l; ++b) {
    *i |= ((k >> (2 * b)) & 1) << b;
    *j |= ((k >> (2 * b + 1)) & 1) << b;
  }
}

static int quad_neighbors(int l, int64_t n, int64_t* out) {
  int64_t i, j, side = (int64_t)1 << l;
  morton_decode(n, l, &i, &j);
  int cnt = 0;
  for (int dj = -1; dj <= 1; ++dj)
    for (int di = -1; di <= 1; ++di) {
      if (di == 0 && dj == 0) continue;
      int64_t a = i + di, b = j + dj;
      if (a < 0 || b < 0 || a >= side || b >= side) continue;
      out[cnt++] = morton_encode(a, b, l);
    }
  return cnt;
}

/* --- septree Neighbors(n, l): N = n (*) {1..6}, keep indices < 7^l --- */
static int sept_neighbors(int l, int64_t n, int64_t* out) {
  int cnt = 0;
  int64_t lim = ipow(7, l);
  for (int d = 1; d <= 6; ++d) {
    int64_t s;
    if (orc_gbt_index_add(n, d, &s) != ORC_OK) continue;
    if (s < lim) out[cnt++] = s;
  }
  return cnt;
}

/* --- triangle-quadtree adjacentNeighbor (Table 1) ---
 * columns k: 0 = Left, 1 = Right, 2 = Vert;  TQ_STAR marks "*" (valid sibling) */
static const int TQ_D[4][3] = {{2, 3, 1}, {3, 2, 0}, {1, 0, 2}, {0, 1, 3}};
static const int TQ_STAR[4][3] = {{1, 1, 1}, {0, 0, 1}, {0, 1, 0}, {1, 0, 0}};

int64_t orc_triq_adjacent(int32_t l, int64_t n, int32_t k) {
  if (n < 0 || l < 1) return -1;
  int t[64];
  for (int i = 1; i <= l; ++i) t[i] = digit_at(n, 4, l, i);
  /* step 1: from right to left, the first valid (starred) entry D[t_i][k] */
  int i = l;
  while (i >= 1 && !TQ_STAR[t[i]][k]) --i;
  if (i < 1) return -1; /* no common ancestor with a sibling in direction k: domain boundary */
  /* step 2: move to the sibling; step 3: reflect the path below the ancestor */
  int orig[64];
  for (int q = 1; q <= l; ++q) orig[q] = t[q];
  t[i] = TQ_D[orig[i]][k];
  for (int j = i + 1; j <= l; ++j) t[j] = TQ_D[orig[j]][k];
  int64_t r = 0;
  for (int q = 1; q <= l; ++q) r = r * 4 + t[q];
  return r;
}

/* Neighbors(n, l) by recursive adjacentNeighbor calls */
static int triq_neighbors(int l, int64_t n, int64_t* out) {
  enum { L_ = 0, R_ = 1, V_ = 2 };
  int64_t Lc = orc_triq_adjacent(l, n, L_), Rc = orc_triq_adjacent(l, n, R_), Vc = orc_triq_adjacent(l, n, V_);
  int64_t VL = orc_triq_adjacent(l, Vc, L_), VR = orc_triq_adjacent(l, Vc, R_);
  int64_t LL = orc_triq_adjacent(l, Lc, L_), RR = orc_triq_adjacent(l, Rc, R_);
  int64_t LV = orc_triq_adjacent(l, Lc, V_), RV = orc_triq_adjacent(l, Rc, V_);
  int64_t VLL = orc_triq_adjacent(l, VL, L_), VRR = orc_triq_adjacent(l, VR, R_);
  int64_t LVR = orc_triq_adjacent(l, LV, R_);
  int64_t all[12] = {Lc, Rc, Vc, VL, VR, LL, RR, LV, RV, VLL, VRR, LVR};
  int cnt = 0;
  for (int a = 0; a < 12; ++a) {
    if (all[a] < 0 || all[a] == n) continue;
    int dup = 0;
    for (int b = 0; b < cnt; ++b) dup |= (out[b] == all[a]);
    if (!dup) out[cnt++] = all[a];
  }
  return cnt;
}

int orc_neighbors(const orc_config* c, int32_t level, int64_t n, int64_t* out) {
  if (level <= 0) return 0; /* the root has no neighbours */
  switch (c->tiling) {
    case ORC_QUAD: return quad_neighbors(level, n, out);
    case ORC_SEPT: return sept_neighbors(level, n, out);
    default: return triq_neighbors(level, n, out);
  }
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static int sort_unique(int64_t* v, int n) {
  qsort(v, (size_t)n, sizeof(int64_t), cmp_i64);
  int k = 0;
  for (int i = 0; i < n; ++i)
    if (k == 0 || v[k - 1] != v[i]) v[k++] = v[i];
  return k;
}

/* NeighborsE4(n, l) = Children[Parent(n) U Neighbors(Parent(n), l-1)]  \  ({n} U Neighbors(n, l))
 * P:104-111 with the set-difference reading D1 (Table 2's P4 = 36-9, 49-7, 52-13). */
int orc_neighbors_e4(const orc_config* c, int32_t level, int64_t n, int64_t* out) {
  int B = branching(c->tiling);
  int64_t par = n / B;
  int64_t pn[16];
  int npn = orc_neighbors(c, level - 1, par, pn);
  int64_t cand[128];
  int nc = 0;
  for (int q = -1; q < npn; ++q) {
    int64_t P = q < 0 ? par : pn[q];
    for (int ch = 0; ch < B; ++ch) cand[nc++] = P * B + ch;
  }
  int64_t near[16];
  int nn = orc_neighbors(c, level, n, near);
  near[nn++] = n;
  int k = 0;
  for (int a = 0; a < nc; ++a) {
    int excl = 0;
    for (int b = 0; b < nn; ++b) excl |= (cand[a] == near[b]);
    if (!excl) out[k++] = cand[a];
  }
  return sort_unique(out, k);
}

/* ======================================================================
 * 3. Spatial addressing: CellCenter / CellIndex
 * ====================================================================== */

/* septree leaf circumradius r = R0 * 7^(-L/2)  (D8), as a fixed IEEE sequence */
static double sept_leaf_r(const orc_config* c) {
  int L = c->depth;
  double den = (double)ipow(7, L / 2);
  if (L % 2) den = den * sqrt(7.0);
  return c->root_size / den;
}

/* lattice coordinates (b, c) of the unit digits 1..6 on the digit-1 / digit-2
 * axes of the lattice of P:230 (D3, D5): unit d at angle d*pi/3 - pi/6. */
static const int UNIT_B[7] = {0, 1, 0, -1, -1, 0, 1};
static const int UNIT_C[7] = {0, 0, 1, 1, 0, -1, -1};

/* integer lattice coordinates of the zero-extended component d 0^k, by the
 * vector form of P:168: v(d0^k) = v(d0^{k-1}) + 2 v([1+(d mod 6)]0^{k-1}) */
static void sept_ze_coords(int d, int k, int64_t* b, int64_t* cc) {
  if (d == 0) {
    *b = 0;
    *cc = 0;
    return;
  }
  if (k == 0) {
    *b = UNIT_B[d];
    *cc = UNIT_C[d];
    return;
  }
  int64_t b1, c1, b2, c2;
  sept_ze_coords(d, k - 1, &b1, &c1);
  sept_ze_coords(1 + (d % 6), k - 1, &b2, &c2);
  *b = b1 + 2 * b2;
  *cc = c1 + 2 * c2;
}

/* CellCenter for the septree: sum of the vectors of the zero-extended
 * components t_i 0^{(|t|-i)+(l_max-l)}, accumulated exactly in lattice units,
 * then mapped to Cartesian by P:230 (D12). */
static void sept_center(const orc_config* c, int l, int64_t n, double* xy) {
  int L = c->depth;
  /* table of v(d 0^k) for the 7 digits and k = 0..L (memo of sept_ze_coords) */
  int64_t ZB[7][24], ZC[7][24];
  for (int k = 0; k <= L; ++k)
    for (int d = 0; d < 7; ++d) {
      if (k == 0 || d == 0) {
        sept_ze_coords(d, 0, &ZB[d][k], &ZC[d][k]);
      } else {
        int e = 1 + (d % 6);
        ZB[d][k] = ZB[d][k - 1] + 2 * ZB[e][k - 1];
        ZC[d][k] = ZC[d][k - 1] + 2 * ZC[e][k - 1];
      }
    }
  int64_t b = 0, cc = 0;
  for (int i = 1; i <= l; ++i) {
    int d = digit_at(n, 7, l, i);
    int k = (l - i) + (L - l);
    b += ZB[d][k];
    cc += ZC[d][k];
  }
  double r = sept_leaf_r(c);
  double A = 1.5 * r, Bc = 0.5 * (S3 * r);
  xy[0] = A * (double)b + c->root_x;
  xy[1] = Bc * (double)(2 * cc + b) + c->root_y;
}

/* triangle CellCenter: sum over components of F(t, i), with
 * theta_i = isUp(t_{1:i}, j)(pi/2 + 2(t_i-1)pi/3), R_i = 2^{l_max-j} r, j = i;
 * cos/sin of the three angles written as exact constants (0,+-1), (-H,-+1/2), (H,-+1/2) (D12) */
int orc_triq_isup(int64_t t, int32_t nd, int32_t l) {
  int zeros = 0;
  for (int i = 1; i <= nd; ++i) zeros += (digit_at(t, 4, nd, i) == 0);
  int parity = zeros % 2;
  int v = (parity + l - nd + 1) % 2;
  if (v < 0) v += 2;
  return 2 * v - 1;
}

static void triq_center(const orc_config* c, int l, int64_t n, double* xy) {
  double x = 0.0, y = 0.0;
  for (int i = 1; i <= l; ++i) {
    int ti = digit_at(n, 4, l, i);
    if (ti == 0) continue; /* "no translations are necessary" */
    int64_t prefix = n / ipow(4, l - i);
    int s = orc_triq_isup(prefix, i, i);
    double Ri = ldexp(c->root_size, -i);
    if (ti == 1) {
      y = y + (double)s * Ri;
    } else if (ti == 2) {
      x = x - Ri * H;
      y = y - (double)s * (0.5 * Ri);
    } else {
      x = x + Ri * H;
      y = y - (double)s * (0.5 * Ri);
    }
  }
  xy[0] = x + c->root_x;
  xy[1] = y + c->root_y;
}

static void quad_center(const orc_config* c, int l, int64_t n, double* xy) {
  int64_t i, j;
  morton_decode(n, l, &i, &j);
  double S = c->root_size;
  xy[0] = c->root_x + S * ldexp((double)(2 * i + 1), -(l + 1));
  xy[1] = c->root_y + S * ldexp((double)(2 * j + 1), -(l + 1));
}

void orc_cell_center(const orc_config* c, int32_t level, int64_t n, double* xy) {
  switch (c->tiling) {
    case ORC_QUAD: quad_center(c, level, n, xy); break;
    case ORC_SEPT: sept_center(c, level, n, xy); break;
    default: triq_center(c, level, n, xy); break;
  }
}

/* literal polar forms, cross-check only (P:192-197 septree, P:326-333 triangle) */
void orc_cell_center_polar(const orc_config* c, int32_t l, int64_t n, double* xy) {
  double x = 0.0, y = 0.0;
  if (c->tiling == ORC_SEPT) {
    double r = sept_leaf_r(c);
    int L = c->depth;
    for (int i = 1; i <= l; ++i) {
      int ti = digit_at(n, 7, l, i);
      if (ti == 0) continue;
      int j = (l - i) + (L - l);
      double th = j * atan(sqrt(3.0) / 2.0) + ti * M_PI / 3.0 - M_PI / 6.0;
      double R = r * sqrt(3.0) * pow(sqrt(7.0), j);
      x += R * cos(th);
      y += R * sin(th);
    }
  } else if (c->tiling == ORC_TRIQ) {
    for (int i = 1; i <= l; ++i) {
      int ti = digit_at(n, 4, l, i);
      if (ti == 0) continue;
      int64_t prefix = n / ipow(4, l - i);
      double th = orc_triq_isup(prefix, i, i) * (M_PI / 2.0 + 2.0 * (ti - 1) * M_PI / 3.0);
      double R = ldexp(c->root_size, -i);
      x += R * cos(th);
      y += R * sin(th);
    }
  } else {
    quad_center(c, l, n, xy);
    return;
  }
  xy[0] = x + c->root_x;
  xy[1] = y + c->root_y;
}

/* --- septree CellIndex --- */
typedef struct {
  int K;           /* axis tables cover -K..K */
  int32_t* dig;    /* [2][2K+1][MAXD] digits */
  int32_t* len;    /* [2][2K+1] */
} sept_axes;

/* u_7 / v_7 of step 5: GBT address of k units along the digit-1 (b) or
 * digit-2 (c) axis (D5), built by repeated table-driven (*) of the unit. */
static int sept_axes_build(const orc_config* c, sept_axes* ax) {
  int L = c->depth;
  ax->K = (int)ceil(1.5 * pow(7.0, L / 2.0)) + 4;
  int W = 2 * ax->K + 1;
  ax->dig = (int32_t*)calloc((size_t)2 * W * MAXD, sizeof(int32_t));
  ax->len = (int32_t*)calloc((size_t)2 * W, sizeof(int32_t));
  if (!ax->dig || !ax->len) return ORC_ENOMEM;
  for (int axis = 0; axis < 2; ++axis) {
    int unit_pos = axis == 0 ? 1 : 2, unit_neg = axis == 0 ? 4 : 5;
    int32_t* d0 = ax->dig + ((size_t)axis * W + ax->K) * MAXD;
    d0[0] = 0;
    ax->len[axis * W + ax->K] = 1;
    for (int s = -1; s <= 1; s += 2) {
      int unit = s > 0 ? unit_pos : unit_neg;
      for (int k = 1; k <= ax->K; ++k) {
        int prev = ax->K + s * (k - 1), cur = ax->K + s * k;
        int32_t* dp = ax->dig + ((size_t)axis * W + prev) * MAXD;
        int32_t* dc = ax->dig + ((size_t)axis * W + cur) * MAXD;
        int32_t u = unit;
        ax->len[axis * W + cur] = orc_gbt_add(dp, ax->len[axis * W + prev], &u, 1, dc);
      }
    }
  }
  return ORC_OK;
}

static void sept_axes_free(sept_axes* ax) {
  free(ax->dig);
  free(ax->len);
}

/* steps 1-6 of P:244-250 for one point; D11 fixes the IEEE sequence and the
 * strict-< first-candidate tie rule.  Returns 0 and the L-digit leaf index, or -1. */
static int sept_key(const orc_config* c, const sept_axes* ax, double r, double x, double y, int64_t* key) {
  double xp = x - c->root_x, yp = y - c->root_y;
  double D3r = 3.0 * r;
  double b = (2.0 * xp) / D3r;           /* eq. P:212 */
  double cc = (yp * S3 - xp) / D3r;
  if (!(fabs(b) <= ax->K - 2) || !(fabs(cc) <= ax->K - 2)) return -1;
  double bf = floor(b), bc = ceil(b), cf = floor(cc), ccl = ceil(cc);
  double cb[4] = {bf, bc, bf, bc}, ccand[4] = {cf, cf, ccl, ccl}; /* eq. P:237 order */
  double A = 1.5 * r, Bc = 0.5 * (S3 * r);
  int best = -1;
  double bestd = 0.0;
  for (int q = 0; q < 4; ++q) {
    double lx = A * cb[q];                       /* eq. P:230 */
    double ly = Bc * (2.0 * ccand[q] + cb[q]);
    double dx = xp - lx, dy = yp - ly;
    double d = dx * dx + dy * dy;
    if (best < 0 || d < bestd) {
      best = q;
      bestd = d;
    }
  }
  int bt = (int)cb[best], ct = (int)ccand[best];
  int W = 2 * ax->K + 1;
  const int32_t* u = ax->dig + ((size_t)0 * W + (ax->K + bt)) * MAXD;
  const int32_t* v = ax->dig + ((size_t)1 * W + (ax->K + ct)) * MAXD;
  int32_t out[MAXD];
  int lo = orc_gbt_add(u, ax->len[0 * W + ax->K + bt], v, ax->len[1 * W + ax->K + ct], out);
  if (lo > c->depth) return -1; /* more than L digits: outside the septree domain (D8) */
  *key = digits7_to_index(out, lo);
  return 0;
}

/* --- triangle CellIndex: level-by-level nearest of 4 lattice points --- */
static int triq_key(const orc_config* c, int level, double x, double y, int64_t* key) {
  double xp = x - c->root_x, yp = y - c->root_y;
  double R0 = c->root_size, eps = 1e-12 * R0, lim = R0 + eps;
  /* closed root triangle with a 1e-12 R0 slack (D11) */
  if (!(yp >= -0.5 * R0 - eps) || !(S3 * xp + yp <= lim) || !(-S3 * xp + yp <= lim)) return -1;
  double u = 0.0, v = 0.0;
  int up = 1;
  int64_t t = 0;
  for (int i = 1; i <= level; ++i) {
    double Ri = ldexp(R0, -i), RH = Ri * H, half = 0.5 * Ri;
    double cu[4] = {u, u, u - RH, u + RH};
    double cv[4] = {v, v + (double)up * Ri, v - (double)up * half, v - (double)up * half};
    int best = -1;
    double bestd = 0.0;
    for (int q = 0; q < 4; ++q) {
      double dx = xp - cu[q], dy = yp - cv[q];
      double d = dx * dx + dy * dy;
      if (best < 0 || d < bestd) {
        best = q;
        bestd = d;
      }
    }
    u = cu[best];
    v = cv[best];
    if (best == 0) up = -up; /* step 4: flip orientation on a centre child */
    t = t * 4 + best;
  }
  *key = t;
  return 0;
}

static int quad_key(const orc_config* c, int level, double x, double y, int64_t* key) {
  double fx = (x - c->root_x) / c->root_size, fy = (y - c->root_y) / c->root_size;
  if (!(fx >= 0.0 && fx <= 1.0 && fy >= 0.0 && fy <= 1.0)) return -1;
  int64_t side = (int64_t)1 << level;
  int64_t i = (int64_t)floor(ldexp(fx, level)), j = (int64_t)floor(ldexp(fy, level));
  if (i == side) i = side - 1; /* closed far edge (D11) */
  if (j == side) j = side - 1;
  *key = morton_encode(i, j, level);
  return 0;
}

int orc_cell_index(const orc_config* c, double x, double y, int32_t level, int64_t* out) {
  int64_t k;
  if (c->tiling == ORC_QUAD) {
    if (quad_key(c, level, x, y, &k)) return ORC_EDOMAIN;
  } else if (c->tiling == ORC_TRIQ) {
    if (triq_key(c, level, x, y, &k)) return ORC_EDOMAIN;
  } else {
    sept_axes ax;
    if (sept_axes_build(c, &ax)) return ORC_ENOMEM;
    int e = sept_key(c, &ax, sept_leaf_r(c), x, y, &k);
    sept_axes_free(&ax);
    if (e) return ORC_EDOMAIN;
    k /= ipow(7, c->depth - level); /* first l components t_{1:l} */
  }
  *out = k;
  return ORC_OK;
}

int orc_keys(const orc_config* c, const double* xy, int64_t n, uint32_t* keys, int64_t* bad) {
  sept_axes ax = {0, NULL, NULL};
  double r = 0.0;
  if (c->tiling == ORC_SEPT) {
    if (sept_axes_build(c, &ax)) return ORC_ENOMEM;
    r = sept_leaf_r(c);
  }
  int64_t first_bad = -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t k = 0;
    int e;
    double x = xy[2 * i], y = xy[2 * i + 1];
    if (c->tiling == ORC_QUAD) e = quad_key(c, c->depth, x, y, &k);
    else if (c->tiling == ORC_TRIQ) e = triq_key(c, c->depth, x, y, &k);
    else e = sept_key(c, &ax, r, x, y, &k);
    if (e) {
#pragma omp critical
      if (first_bad < 0 || i < first_bad) first_bad = i;
      keys[i] = 0xffffffffu;
    } else {
      keys[i] = (uint32_t)k;
    }
  }
  if (c->tiling == ORC_SEPT) sept_axes_free(&ax);
  if (first_bad >= 0) {
    if (bad) *bad = first_bad;
    return ORC_EDOMAIN;
  }
  return ORC_OK;
}

/* ======================================================================
 * 4. Operators (classical GR 2D log-kernel forms; D10)
 * ====================================================================== */

static double BINOM[130][130];
static int binom_ready = 0;
static void binom_init(void) {
  if (binom_ready) return;
#pragma omp critical
  {
    if (!binom_ready) {
      for (int n = 0; n < 130; ++n) {
        BINOM[n][0] = 1.0;
        for (int k = 1; k <= n; ++k) BINOM[n][k] = BINOM[n - 1][k - 1] + (k < n ? BINOM[n - 1][k] : 0.0);
      }
      binom_ready = 1;
    }
  }
}

/* principal Log with Arg in (-pi, pi] and a zero imaginary part canonicalised to +0 (D13) */
static cplx c_log(double dx, double dy) {
  if (dy == 0.0) dy = 0.0;
  return log(hypot(dx, dy)) + I * atan2(dy, dx);
}
void orc_log(double dx, double dy, double* out) {
  cplx z = c_log(dx, dy);
  out[0] = creal(z);
  out[1] = cimag(z);
}

/* P2M about c: Q = sum u_i, a_k = -(1/k) sum u_i (x_i - c)^k  (B.2) */
static void p2m_c(const double* xy, const double* u, const int32_t* idx, int64_t n, const double* c, int p, cplx* mp) {
  for (int k = 0; k <= p; ++k) mp[k] = 0.0;
  cplx S[130];
  for (int k = 0; k <= p; ++k) S[k] = 0.0;
  for (int64_t q = 0; q < n; ++q) {
    int64_t i = idx ? idx[q] : q;
    cplx z = (xy[2 * i] - c[0]) + I * (xy[2 * i + 1] - c[1]);
    cplx zk = 1.0;
    S[0] += u[i];
    for (int k = 1; k <= p; ++k) {
      zk = zk * z;
      S[k] += u[i] * zk;
    }
  }
  mp[0] = S[0];
  for (int k = 1; k <= p; ++k) mp[k] = -S[k] / (double)k;
}

/* M2M child -> parent, z0 = c_child - c_parent (B.3):
 *   a'_l = -Q z0^l / l + sum_{k=1..l} a_k z0^{l-k} C(l-1, k-1)                     */
static void m2m_c(const cplx* a, const double* cc, const double* cp, int p, cplx* acc) {
  binom_init();
  cplx z0 = (cc[0] - cp[0]) + I * (cc[1] - cp[1]);
  cplx zp[130];
  zp[0] = 1.0;
  for (int k = 1; k <= p; ++k) zp[k] = zp[k - 1] * z0;
  acc[0] += a[0];
  for (int l = 1; l <= p; ++l) {
    cplx s = -a[0] * zp[l] / (double)l;
    for (int k = 1; k <= l; ++k) s += a[k] * zp[l - k] * BINOM[l - 1][k - 1];
    acc[l] += s;
  }
}

/* M2L, multipole at c_m -> local at c_l, z0 = c_m - c_l (B.4):
 *   b_0 = Q Log(c_l - c_m) + sum_k (-1)^k a_k / z0^k
 *   b_l = -Q / (l z0^l) + z0^{-l} sum_k (-1)^k C(l+k-1, k-1) a_k / z0^k               */
static void m2l_c(const cplx* a, const double* cm, const double* cl, int p, cplx* acc) {
  binom_init();
  cplx z0 = (cm[0] - cl[0]) + I * (cm[1] - cl[1]);
  cplx w = 1.0 / z0;
  cplx wp[130], t[130];
  wp[0] = 1.0;
  for (int k = 1; k <= p; ++k) wp[k] = wp[k - 1] * w;
  for (int k = 1; k <= p; ++k) t[k] = ((k % 2) ? -1.0 : 1.0) * a[k] * wp[k]; /* (-1)^k a_k / z0^k */
  cplx b0 = a[0] * c_log(cl[0] - cm[0], cl[1] - cm[1]);                  /* D13 (iii) */
  for (int k = 1; k <= p; ++k) b0 += t[k];
  acc[0] += b0;
  for (int l = 1; l <= p; ++l) {
    cplx s = 0.0;
    for (int k = 1; k <= p; ++k) s += BINOM[l + k - 1][k - 1] * t[k];
    acc[l] += -a[0] * wp[l] / (double)l + wp[l] * s;
  }
}

/* L2L parent -> child, w = c_child - c_parent (B.5): b'_l = sum_{k=l..p} b_k C(k,l) w^{k-l} */
static void l2l_c(const cplx* b, const double* cp, const double* cc, int p, cplx* out) {
  binom_init();
  cplx w = (cc[0] - cp[0]) + I * (cc[1] - cp[1]);
  cplx wp[130];
  wp[0] = 1.0;
  for (int k = 1; k <= p; ++k) wp[k] = wp[k - 1] * w;
  for (int l = 0; l <= p; ++l) {
    cplx s = 0.0;
    for (int k = l; k <= p; ++k) s += b[k] * BINOM[k][l] * wp[k - l];
    out[l] = s;
  }
}

/* L2P: sum_{l=0..p} b_l (y - c)^l, Horner (B.6) */
static cplx l2p_c(const cplx* b, const double* c, int p, double yx, double yy) {
  cplx z = (yx - c[0]) + I * (yy - c[1]);
  cplx acc = b[p];
  for (int l = p - 1; l >= 0; --l) acc = acc * z + b[l];
  return acc;
}

void orc_p2m(const double* xy, const double* u, int64_t n, const double* c, int32_t p, double* mp) {
  p2m_c(xy, u, NULL, n, c, p, (cplx*)mp);
}
void orc_m2m(const double* mp_child, const double* c_child, const double* c_parent, int32_t p, double* acc) {
  m2m_c((const cplx*)mp_child, c_child, c_parent, p, (cplx*)acc);
}
void orc_m2l(const double* mp, const double* c_m, const double* c_l, int32_t p, double* acc) {
  m2l_c((const cplx*)mp, c_m, c_l, p, (cplx*)acc);
}
void orc_l2l(const double* lp, const double* cp, const double* cc, int32_t p, double* out) {
  l2l_c((const cplx*)lp, cp, cc, p, (cplx*)out);
}
void orc_l2p(const double* loc, const double* c, int32_t p, const double* y, double* phi) {
  cplx v = l2p_c((const cplx*)loc, c, p, y[0], y[1]);
  phi[0] = creal(v);
  phi[1] = cimag(v);
}

/* ======================================================================
 * 5. Direct summation: Phi_j = sum_i u_i Log(y_j - x_i), source order
 * ====================================================================== */
int orc_direct(const double* sxy, const double* u, int64_t n, const double* txy, int64_t m, int32_t self_mode,
               const int64_t* tgt_ids, int64_t ntgt, double* phi, int64_t* bad) {
  if (!tgt_ids) ntgt = m;
  int64_t first_bad = -1;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < ntgt; ++q) {
    int64_t j = tgt_ids ? tgt_ids[q] : q;
    double yx = txy[2 * j], yy = txy[2 * j + 1];
    cplx s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      if (self_mode && i == j) continue; /* D16 */
      double dx = yx - sxy[2 * i], dy = yy - sxy[2 * i + 1];
      if (dx == 0.0 && dy == 0.0) {
#pragma omp critical
        if (first_bad < 0 || j < first_bad) first_bad = j;
        continue;
      }
      s += u[i] * c_log(dx, dy);
    }
    phi[2 * q] = creal(s);
    phi[2 * q + 1] = cimag(s);
  }
  if (first_bad >= 0) {
    if (bad) *bad = first_bad;
    return ORC_ECOINCIDENT;
  }
  return ORC_OK;
}

/* ======================================================================
 * 6. The FMM tree (SURVEY §8(c) algorithm, steps 1-8)
 * ====================================================================== */
struct orc_tree {
  orc_config cfg;
  int B, L, p;
  int64_t n, m;
  double *sxy, *su, *txy;        /* copies of the inputs (input order) */
  uint32_t *skey, *tkey;         /* leaf keys, input order */
  int32_t *sperm, *tperm;        /* sorted position -> input index */
  int64_t *soff, *toff;          /* leaf CSR over sorted order, K+1 */
  int64_t **scnt, **tcnt;        /* per-level occupancy [l][cell], l = 0..L */
  double** cen;                  /* per-level centres [l][2*cell], l = 0..L (computed lazily) */
  cplx** mp;                     /* per-level multipoles [l][cell*(p+1)] */
  cplx** loc;                    /* per-level locals */
  uint8_t** loc_done;
  double* absu_prefix;           /* prefix sums of |u| in sorted order (bound) */
  int upward_done;
};

typedef struct {
  uint32_t key;
  int32_t idx;
} keyidx;
static int cmp_keyidx(const void* a, const void* b) {
  const keyidx *x = a, *y = b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

/* step 3: sort by (key, original index) and build the leaf CSR ("order relation in memory") */
static int sort_and_csr(const uint32_t* key, int64_t n, int64_t K, int32_t* perm, int64_t* off) {
  keyidx* ki = (keyidx*)malloc(sizeof(keyidx) * (size_t)(n > 0 ? n : 1));
  if (!ki) return ORC_ENOMEM;
  for (int64_t i = 0; i < n; ++i) {
    ki[i].key = key[i];
    ki[i].idx = (int32_t)i;
  }
  qsort(ki, (size_t)n, sizeof(keyidx), cmp_keyidx);
  for (int64_t i = 0; i <= K; ++i) off[i] = 0;
  for (int64_t i = 0; i < n; ++i) {
    perm[i] = ki[i].idx;
    off[ki[i].key + 1]++;
  }
  for (int64_t i = 0; i < K; ++i) off[i + 1] += off[i];
  free(ki);
  return ORC_OK;
}

void orc_tree_free(orc_tree* t) {
  if (!t) return;
  free(t->sxy); free(t->su); free(t->txy);
  free(t->skey); free(t->tkey); free(t->sperm); free(t->tperm);
  free(t->soff); free(t->toff); free(t->absu_prefix);
  for (int l = 0; l <= t->L; ++l) {
    if (t->scnt) free(t->scnt[l]);
    if (t->tcnt) free(t->tcnt[l]);
    if (t->cen) free(t->cen[l]);
    if (t->mp) free(t->mp[l]);
    if (t->loc) free(t->loc[l]);
    if (t->loc_done) free(t->loc_done[l]);
  }
  free(t->scnt); free(t->tcnt); free(t->cen); free(t->mp); free(t->loc); free(t->loc_done);
  free(t);
}

int orc_tree_build(const orc_config* c, const double* sxy, const double* u, int64_t n, const double* txy,
                   int64_t m, orc_tree** out, int64_t* bad) {
  if (c->depth < 1 || c->p < 1 || c->p > 64 || !(c->root_size > 0.0)) return ORC_EBADCFG;
  if (c->tiling == ORC_SEPT && c->depth > 10) return ORC_EBADCFG;
  if (c->tiling != ORC_SEPT && c->depth > 15) return ORC_EBADCFG;
  if (c->tiling < 0 || c->tiling > 2) return ORC_EBADCFG;
  if (c->self_mode) {
    txy = sxy;
    m = n;
  }
  orc_tree* t = (orc_tree*)calloc(1, sizeof(orc_tree));
  if (!t) return ORC_ENOMEM;
  t->cfg = *c;
  t->B = branching(c->tiling);
  t->L = c->depth;
  t->p = c->p;
  t->n = n;
  t->m = m;
  int64_t K = ipow(t->B, t->L);
  size_t nn = (size_t)(n > 0 ? n : 1), mm = (size_t)(m > 0 ? m : 1);
  t->sxy = malloc(16 * nn); t->su = malloc(8 * nn); t->txy = malloc(16 * mm);
  t->skey = malloc(4 * nn); t->tkey = malloc(4 * mm);
  t->sperm = malloc(4 * nn); t->tperm = malloc(4 * mm);
  t->soff = malloc(8 * (size_t)(K + 1)); t->toff = malloc(8 * (size_t)(K + 1));
  t->absu_prefix = malloc(8 * (nn + 1));
  t->scnt = calloc((size_t)t->L + 1, sizeof(int64_t*)); t->tcnt = calloc((size_t)t->L + 1, sizeof(int64_t*));
  t->cen = calloc((size_t)t->L + 1, sizeof(double*));
  t->mp = calloc((size_t)t->L + 1, sizeof(cplx*)); t->loc = calloc((size_t)t->L + 1, sizeof(cplx*));
  t->loc_done = calloc((size_t)t->L + 1, sizeof(uint8_t*));
  if (!t->sxy || !t->su || !t->txy || !t->skey || !t->tkey || !t->sperm || !t->tperm || !t->soff || !t->toff ||
      !t->absu_prefix || !t->scnt || !t->tcnt || !t->cen || !t->mp || !t->loc || !t->loc_done) {
    orc_tree_free(t);
    return ORC_ENOMEM;
  }
  if (n) memcpy(t->sxy, sxy, 16 * (size_t)n);
  if (n) memcpy(t->su, u, 8 * (size_t)n);
  if (m) memcpy(t->txy, txy, 16 * (size_t)m);
  /* step 2: keying (CellIndex at the leaf level) */
  int64_t b = -1;
  int e = orc_keys(c, t->sxy, n, t->skey, &b);
  if (e == ORC_OK && !c->self_mode) e = orc_keys(c, t->txy, m, t->tkey, &b);
  if (e == ORC_OK && c->self_mode && m) memcpy(t->tkey, t->skey, 4 * (size_t)m);
  if (e != ORC_OK) {
    if (bad) *bad = b;
    orc_tree_free(t);
    return e;
  }
  /* step 3: stable sort + leaf CSR */
  if (sort_and_csr(t->skey, n, K, t->sperm, t->soff) || sort_and_csr(t->tkey, m, K, t->tperm, t->toff)) {
    orc_tree_free(t);
    return ORC_ENOMEM;
  }
  t->absu_prefix[0] = 0.0;
  for (int64_t q = 0; q < n; ++q) t->absu_prefix[q + 1] = t->absu_prefix[q] + fabs(t->su[t->sperm[q]]);
  /* per-level occupancy: leaves from the CSR, parents = sum of children */
  for (int l = t->L; l >= 0; --l) {
    int64_t nc = ipow(t->B, l);
    t->scnt[l] = malloc(8 * (size_t)nc);
    t->tcnt[l] = malloc(8 * (size_t)nc);
    if (!t->scnt[l] || !t->tcnt[l]) {
      orc_tree_free(t);
      return ORC_ENOMEM;
    }
    for (int64_t cidx = 0; cidx < nc; ++cidx) {
      if (l == t->L) {
        t->scnt[l][cidx] = t->soff[cidx + 1] - t->soff[cidx];
        t->tcnt[l][cidx] = t->toff[cidx + 1] - t->toff[cidx];
      } else {
        int64_t s = 0, q = 0;
        for (int ch = 0; ch < t->B; ++ch) {
          s += t->scnt[l + 1][cidx * t->B + ch];
          q += t->tcnt[l + 1][cidx * t->B + ch];
        }
        t->scnt[l][cidx] = s;
        t->tcnt[l][cidx] = q;
      }
    }
  }
  *out = t;
  return ORC_OK;
}

void orc_tree_keys(const orc_tree* t, uint32_t* sk, uint32_t* tk) {
  if (sk && t->n) memcpy(sk, t->skey, 4 * (size_t)t->n);
  if (tk && t->m) memcpy(tk, t->tkey, 4 * (size_t)t->m);
}
void orc_tree_perm(const orc_tree* t, int32_t* sp, int32_t* tp) {
  if (sp && t->n) memcpy(sp, t->sperm, 4 * (size_t)t->n);
  if (tp && t->m) memcpy(tp, t->tperm, 4 * (size_t)t->m);
}
void orc_tree_leaf_offsets(const orc_tree* t, int64_t* so, int64_t* to) {
  int64_t K = ipow(t->B, t->L);
  if (so) memcpy(so, t->soff, 8 * (size_t)(K + 1));
  if (to) memcpy(to, t->toff, 8 * (size_t)(K + 1));
}
int64_t orc_tree_count(const orc_tree* t, int32_t l, int64_t cell, int32_t which) {
  return which ? t->tcnt[l][cell] : t->scnt[l][cell];
}

/* step 5: near(t) = ({t} U Neighbors(t, L)) restricted to non-empty source leaves, ascending */
int orc_tree_near(const orc_tree* t, int64_t leaf, int64_t* out) {
  int64_t nb[16];
  int k = orc_neighbors(&t->cfg, t->L, leaf, nb);
  nb[k++] = leaf;
  int q = 0;
  for (int a = 0; a < k; ++a)
    if (t->scnt[t->L][nb[a]] > 0) out[q++] = nb[a];
  return sort_unique(out, q);
}

/* step 5: E4 at level l restricted to non-empty source cells (D1, D2, D17) */
int orc_tree_e4(const orc_tree* t, int32_t l, int64_t cell, int64_t* out) {
  int64_t all[128];
  int k = orc_neighbors_e4(&t->cfg, l, cell, all);
  int q = 0;
  for (int a = 0; a < k; ++a)
    if (t->scnt[l][all[a]] > 0) out[q++] = all[a];
  return q;
}

/* canonical CSR of near (level < 0) or E4 (level l) lists over non-empty target cells */
static int lists_csr(const orc_tree* t, int l, int32_t* owners, int64_t* offs, int32_t* entries, int64_t* nown,
                     int64_t* nent) {
  int level = l < 0 ? t->L : l;
  int64_t nc = ipow(t->B, level), no = 0, ne = 0;
  int64_t buf[128];
  if (offs) offs[0] = 0;
  for (int64_t c = 0; c < nc; ++c) {
    if (t->tcnt[level][c] == 0) continue;
    int k = l < 0 ? orc_tree_near(t, c, buf) : orc_tree_e4(t, level, c, buf);
    if (owners) owners[no] = (int32_t)c;
    for (int a = 0; a < k; ++a) {
      if (entries) entries[ne] = (int32_t)buf[a];
      ++ne;
    }
    ++no;
    if (offs) offs[no] = ne;
  }
  *nown = no;
  *nent = ne;
  return ORC_OK;
}
int orc_tree_near_csr(const orc_tree* t, int32_t* owners, int64_t* offs, int32_t* entries, int64_t* nown,
                      int64_t* nent) {
  return lists_csr(t, -1, owners, offs, entries, nown, nent);
}
int orc_tree_e4_csr(const orc_tree* t, int32_t level, int32_t* owners, int64_t* offs, int32_t* entries,
                    int64_t* nown, int64_t* nent) {
  if (level < 1 || level > t->L) return ORC_EBADCFG;
  return lists_csr(t, level, owners, offs, entries, nown, nent);
}

static const double* centre_of(orc_tree* t, int l, int64_t cell);
void orc_tree_centres(orc_tree* t, int32_t level, double* xy) {
  const double* c = centre_of(t, level, 0);
  memcpy(xy, c, 16 * (size_t)ipow(t->B, level));
}

static const double* centre_of(orc_tree* t, int l, int64_t cell) {
  if (!t->cen[l]) {
#pragma omp critical
    if (!t->cen[l]) {
      int64_t nc = ipow(t->B, l);
      double* cen = malloc(16 * (size_t)nc);
      for (int64_t q = 0; q < nc; ++q) orc_cell_center(&t->cfg, l, q, cen + 2 * q);
      t->cen[l] = cen;
    }
  }
  return t->cen[l] + 2 * cell;
}

/* step 6: P2M at non-empty source leaves, M2M for l = L-1..1, children ascending */
void orc_tree_upward(orc_tree* t) {
  if (t->upward_done) return;
  int p = t->p, L = t->L;
  for (int l = 0; l <= L; ++l) {
    centre_of(t, l, 0);
    int64_t nc = ipow(t->B, l);
    t->mp[l] = calloc((size_t)nc * (size_t)(p + 1), sizeof(cplx));
  }
  int64_t K = ipow(t->B, L);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t leaf = 0; leaf < K; ++leaf) {
    int64_t s0 = t->soff[leaf], s1 = t->soff[leaf + 1];
    if (s1 == s0) continue;
    p2m_c(t->sxy, t->su, t->sperm + s0, s1 - s0, t->cen[L] + 2 * leaf, p, t->mp[L] + leaf * (p + 1));
  }
  for (int l = L - 1; l >= 1; --l) {
    int64_t nc = ipow(t->B, l);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t cidx = 0; cidx < nc; ++cidx) {
      if (t->scnt[l][cidx] == 0) continue;
      for (int ch = 0; ch < t->B; ++ch) {
        int64_t child = cidx * t->B + ch;
        if (t->scnt[l + 1][child] == 0) continue;
        m2m_c(t->mp[l + 1] + child * (p + 1), t->cen[l + 1] + 2 * child, t->cen[l] + 2 * cidx, p,
              t->mp[l] + cidx * (p + 1));
      }
    }
  }
  t->upward_done = 1;
}

void orc_tree_multipoles_level(orc_tree* t, int32_t l, double* mp) {
  orc_tree_upward(t);
  memcpy(mp, t->mp[l], sizeof(cplx) * (size_t)(t->p + 1) * (size_t)ipow(t->B, l));
}

void orc_tree_multipole(const orc_tree* t, int32_t l, int64_t cell, double* mp) {
  memcpy(mp, t->mp[l] + cell * (t->p + 1), sizeof(cplx) * (size_t)(t->p + 1));
}

/* step 7 for one cell: L2L from the parent (l >= 2), then M2L over E4 ascending */
static int64_t compute_local(orc_tree* t, int l, int64_t cell) {
  int p = t->p;
  cplx* b = t->loc[l] + cell * (p + 1);
  if (l >= 2) {
    int64_t par = cell / t->B;
    l2l_c(t->loc[l - 1] + par * (p + 1), t->cen[l - 1] + 2 * par, t->cen[l] + 2 * cell, p, b);
  } else {
    for (int k = 0; k <= p; ++k) b[k] = 0.0;
  }
  int64_t e4[128];
  int ne = orc_tree_e4(t, l, cell, e4);
  for (int q = 0; q < ne; ++q)
    m2l_c(t->mp[l] + e4[q] * (p + 1), t->cen[l] + 2 * e4[q], t->cen[l] + 2 * cell, p, b);
  return ne;
}

/* make sure the locals of the leaves of the given targets and of all their
 * ancestors exist; level by level, cells in ascending order (parallel over cells) */
static int64_t ensure_locals(orc_tree* t, const int64_t* tgt_ids, int64_t ntgt) {
  int L = t->L, p = t->p;
  orc_tree_upward(t);
  for (int l = 0; l <= L; ++l)
    if (!t->loc[l]) {
      int64_t nc = ipow(t->B, l);
      t->loc[l] = calloc((size_t)nc * (size_t)(p + 1), sizeof(cplx));
      t->loc_done[l] = calloc((size_t)nc, 1);
    }
  /* mark needed cells */
  uint8_t** need = calloc((size_t)L + 1, sizeof(uint8_t*));
  for (int l = 1; l <= L; ++l) need[l] = calloc((size_t)ipow(t->B, l), 1);
  if (!tgt_ids) ntgt = t->m;
  for (int64_t q = 0; q < ntgt; ++q) {
    int64_t j = tgt_ids ? tgt_ids[q] : q;
    int64_t cell = t->tkey[j];
    for (int l = L; l >= 1; --l) {
      need[l][cell] = 1;
      cell /= t->B;
    }
  }
  int64_t m2l_ops = 0;
  for (int l = 1; l <= L; ++l) {
    int64_t nc = ipow(t->B, l);
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : m2l_ops)
    for (int64_t cidx = 0; cidx < nc; ++cidx) {
      if (!need[l][cidx] || t->loc_done[l][cidx]) continue;
      m2l_ops += compute_local(t, l, cidx);
      t->loc_done[l][cidx] = 1;
    }
  }
  for (int l = 1; l <= L; ++l) free(need[l]);
  free(need);
  return m2l_ops;
}

void orc_tree_local(orc_tree* t, int32_t l, int64_t cell, double* loc) {
  /* find any target below this cell to drive ensure_locals; else compute directly */
  if (!t->loc[l] || !t->loc_done[l][cell]) {
    int64_t leaf0 = cell * ipow(t->B, t->L - l), leaf1 = (cell + 1) * ipow(t->B, t->L - l);
    int64_t tj = -1;
    for (int64_t q = t->toff[leaf0]; q < t->toff[leaf1] && tj < 0; ++q) tj = t->tperm[q];
    if (tj >= 0) ensure_locals(t, &tj, 1);
  }
  if (t->loc[l] && t->loc_done[l][cell])
    memcpy(loc, t->loc[l] + cell * (t->p + 1), sizeof(cplx) * (size_t)(t->p + 1));
  else
    memset(loc, 0, sizeof(cplx) * (size_t)(t->p + 1));
}

/* step 8: Phi_j = L2P(local of leaf(j)) + sum over near leaves (ascending) of
 * sources (sorted order) of u_i Log(y_j - x_i), skipping i == j in self mode */
int orc_tree_evaluate(orc_tree* t, const int64_t* tgt_ids, int64_t ntgt, double* phi, int64_t* bad,
                      int64_t* counters) {
  int L = t->L, p = t->p;
  int64_t m2l_ops = ensure_locals(t, tgt_ids, ntgt);
  if (!tgt_ids) ntgt = t->m;
  int64_t first_bad = -1, pairs = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : pairs)
  for (int64_t q = 0; q < ntgt; ++q) {
    int64_t j = tgt_ids ? tgt_ids[q] : q;
    int64_t leaf = t->tkey[j];
    double yx = t->txy[2 * j], yy = t->txy[2 * j + 1];
    cplx far = l2p_c(t->loc[L] + leaf * (p + 1), t->cen[L] + 2 * leaf, p, yx, yy);
    cplx near = 0.0;
    int64_t nl[16];
    int nn = orc_tree_near(t, leaf, nl);
    for (int a = 0; a < nn; ++a) {
      for (int64_t s = t->soff[nl[a]]; s < t->soff[nl[a] + 1]; ++s) {
        int64_t i = t->sperm[s];
        if (t->cfg.self_mode && i == j) continue;
        double dx = yx - t->sxy[2 * i], dy = yy - t->sxy[2 * i + 1];
        if (dx == 0.0 && dy == 0.0) {
#pragma omp critical
          if (first_bad < 0 || j < first_bad) first_bad = j;
          continue;
        }
        near += t->su[i] * c_log(dx, dy);
        ++pairs;
      }
    }
    cplx v = far + near;
    phi[2 * q] = creal(v);
    phi[2 * q + 1] = cimag(v);
  }
  if (counters) {
    counters[0] = m2l_ops;
    counters[1] = pairs;
  }
  if (first_bad >= 0) {
    if (bad) *bad = first_bad;
    return ORC_ECOINCIDENT;
  }
  return ORC_OK;
}

/* D14: B_j = sum_l sum_{s in E4_l(anc_l(j))} (A_s / rho_l) (1/(1+rho/r))^{p+1},
 * rho_l = (rho/r) r_l with Table 2's rho/r and the idealised level
 * circumradius r_l (M2L bound of P:403). */
void orc_tree_bound(orc_tree* t, const int64_t* tgt_ids, int64_t ntgt, double* bound) {
  int L = t->L, p = t->p;
  double rho_over_r, rL;
  if (t->cfg.tiling == ORC_QUAD) {
    rho_over_r = 2.0 * (sqrt(2.0) - 1.0);
    rL = t->cfg.root_size * ldexp(1.0, -L) / sqrt(2.0);
  } else if (t->cfg.tiling == ORC_SEPT) {
    rho_over_r = 1.0;
    rL = sept_leaf_r(&t->cfg);
  } else {
    rho_over_r = sqrt(7.0) - 2.0;
    rL = ldexp(t->cfg.root_size, -L);
  }
  double fac = pow(1.0 / (1.0 + rho_over_r), p + 1);
  if (!tgt_ids) ntgt = t->m;
  for (int64_t q = 0; q < ntgt; ++q) {
    int64_t j = tgt_ids ? tgt_ids[q] : q;
    int64_t cell = t->tkey[j];
    double Bj = 0.0;
    for (int l = L; l >= 1; --l) {
      double rl = (t->cfg.tiling == ORC_SEPT) ? rL * pow(sqrt(7.0), L - l) : rL * ldexp(1.0, L - l);
      double rho = rho_over_r * rl;
      int64_t e4[128];
      int ne = orc_tree_e4(t, l, cell, e4);
      int64_t span = ipow(t->B, L - l);
      for (int a = 0; a < ne; ++a) {
        int64_t s0 = t->soff[e4[a] * span], s1 = t->soff[(e4[a] + 1) * span];
        double As = t->absu_prefix[s1] - t->absu_prefix[s0];
        Bj += As / rho * fac;
      }
      cell /= t->B;
    }
    bound[q] = Bj;
  }
}

/* ------------------------------------------------------------------ cost model (NEXT-2)
 * Appendices A-C, eqs. app:quadbefore / app:sepbefore / app:tquadbefore:
 *   cost(FMM) = (M + N) P + (K B/(B-1) (P4 + 2) - C0) P^2 + M (P2 s + P),
 *   K = B^L leaves, s = N / K points per leaf, (B, P4, P2) = (4, 27, 9), (7, 42, 7), (4, 39, 13)
 * (Table 2).  C0 does not depend on L (and is garbled for the triangle tree, reading
 * D19), so it is left out: it does not move the minimum over L. */
static void orc_cost_params(int tiling, double* B, double* P4, double* P2) {
  if (tiling == ORC_QUAD) {
    *B = 4.0; *P4 = 27.0; *P2 = 9.0;
  } else if (tiling == ORC_SEPT) {
    *B = 7.0; *P4 = 42.0; *P2 = 7.0;
  } else {
    *B = 4.0; *P4 = 39.0; *P2 = 13.0;
  }
}

double orc_paper_cost(int tiling, double n, double m, int p, int depth) {
  double B, P4, P2;
  orc_cost_params(tiling, &B, &P4, &P2);
  double K = pow(B, depth), s = n / K, P = (double)p;
  return (m + n) * P + K * B / (B - 1.0) * (P4 + 2.0) * P * P + m * (P2 * s + P);
}

/* the depth 1..maxdepth of least paper cost (the first one on ties) */
int orc_paper_depth(int tiling, double n, double m, int p, int maxdepth) {
  int best = 1;
  double bc = orc_paper_cost(tiling, n, m, p, 1);
  for (int L = 2; L <= maxdepth; ++L) {
    double c = orc_paper_cost(tiling, n, m, p, L);
    if (c < bc) {
      bc = c;
      best = L;
    }
  }
  return best;
}

/* ======================================================================
 * 7. NEXT-4: regular-polygon point picking (Fig. 12; reading D22)
 *
 * "the polygon is subdivided into disjoint isosceles triangles per edge where halves of
 * triangles are rearranged to form rectangles.  Uniformly random points (x,y) are picked
 * from this rectangle and a third uniformly random variable z assigns the point to one of
 * the isosceles triangles".  The random numbers are counter-based (D22): draw d of
 * point g is h(seed, 4g + d), the SplitMix64 output after 4g + d + 1 increments of the
 * state `seed`, so any point can be drawn alone (sampled parity checks, rank slices).
 * ====================================================================== */
uint64_t orc_draw(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double unit53(uint64_t h) { return (double)(h >> 11) * 0x1p-53; } /* [0, 1), 53 bits */

/* cos and sin of k pi / 6, k = 0..11, exact where the value is 0, 1/2 or 1 (H otherwise) */
static void dir_pi6(int k, double* c, double* s) {
  static const double C[12] = {1.0, H, 0.5, 0.0, -0.5, -H, -1.0, -H, -0.5, 0.0, 0.5, H};
  *c = C[k % 12];
  *s = C[(k + 9) % 12]; /* sin(k pi/6) = cos((k - 3) pi/6) */
}

int orc_sample_cells(const orc_config* c, const int64_t* cells, int64_t ncells, int32_t per_cell, uint64_t seed,
                     int64_t first, double* xy, double* u) {
  const int L = c->depth;
  const int64_t K = ipow(c->tiling == ORC_SEPT ? 7 : 4, L);
  /* polygon of a leaf: nsides, half-edge a, apothem b (the rectangle is a x b) */
  int nsides;
  double a, b;
  if (c->tiling == ORC_QUAD) { /* square of side S 2^-L */
    nsides = 4;
    a = 0.5 * ldexp(c->root_size, -L);
    b = a;
  } else if (c->tiling == ORC_SEPT) { /* hexagon of circumradius r (D8), a vertex at angle 0 */
    nsides = 6;
    double r = sept_leaf_r(c);
    a = 0.5 * r;
    b = H * r;
  } else { /* triangle of circumradius R0 2^-L, upright or inverted (isUp) */
    nsides = 3;
    double R = ldexp(c->root_size, -L);
    a = H * R;
    b = 0.5 * R;
  }
  for (int64_t i = 0; i < ncells; ++i) {
    int64_t cell = cells ? cells[i] : i;
    if (cell < 0 || cell >= K) return ORC_EDOMAIN;
    double cen[2];
    orc_cell_center(c, L, cell, cen);
    /* apothem direction of edge z, in units of pi/6:
     *   quad 3z (edges facing 0, pi/2, pi, 3pi/2), hexagon 2z + 1 (pi/6 + z pi/3),
     *   upright triangle 4z + 1 (pi/6, 5pi/6, 3pi/2), inverted 4z + 3 (pi/2, 7pi/6, 11pi/6) */
    int step = c->tiling == ORC_QUAD ? 3 : (c->tiling == ORC_SEPT ? 2 : 4);
    int off = c->tiling == ORC_QUAD ? 0 : (c->tiling == ORC_SEPT ? 1 : (orc_triq_isup(cell, L, L) > 0 ? 1 : 3));
    for (int32_t j = 0; j < per_cell; ++j) {
      const int64_t o = i * per_cell + j;
      const uint64_t g = (uint64_t)(first + o);
      const double s = unit53(orc_draw(seed, 4 * g + 0));
      const double t = unit53(orc_draw(seed, 4 * g + 1));
      const int z = (int)(((orc_draw(seed, 4 * g + 2) >> 32) * (uint64_t)nsides) >> 32);
      /* rectangle [0, a] x [0, b]: the half s <= t is the right half of the isosceles
       * triangle (X along the edge, Y along the apothem), the half s > t is moved onto its
       * left half */
      double X, Y;
      if (s > t) {
        X = (s - 1.0) * a;
        Y = (1.0 - t) * b;
      } else {
        X = s * a;
        Y = t * b;
      }
      double cs, sn;
      dir_pi6(step * z + off, &cs, &sn);
      /* rotate: +Y along the apothem direction (cs, sn), +X along (sn, -cs) */
      const double px = Y * cs + X * sn;
      const double py = Y * sn - X * cs;
      xy[2 * o] = cen[0] + px;
      xy[2 * o + 1] = cen[1] + py;
      if (u) u[o] = 2.0 * unit53(orc_draw(seed, 4 * g + 3)) - 1.0;
    }
  }
  return ORC_OK;
}
