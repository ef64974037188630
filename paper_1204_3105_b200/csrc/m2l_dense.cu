// m2l_dense.cu -- SURVEY §8(f) NEXT-3: M2L with precomputed per-offset operators (the paper names
// its on-the-fly translation matrices as its inefficiency), on the FP64 tensor cores.
//
// Quadtree levels l >= 2.  Every interior cell t at level l has 27 E4 sources (Table 2 P4,
// P:413-415), at offsets d = s - t in {-2-cx .. 3-cx} x {-2-cy .. 3-cy} minus the 3 x 3 near
// block, where (cx, cy) is t's child position (Morton digit, D7).  The quadtree centres are
// exact binary fractions of the root side (D12), so every pair with the same offset has the same
// z0 = c_s - c_t = h (dx + i dy), h = S 2^-l, and the whole M2L (App. B.4, including
// b_0's Q Log(c_t - c_s) on the canonical branch, D13) is one complex (p+1) x (p+1) matrix T_d:
//   T[0][0] = Log(-z0), T[0][k] = (-1)^k w^k, T[l][0] = -w^l / l, T[l][k] = C(l+k-1, k-1) (-1)^k w^(l+k),
// w = 1 / z0.  The 7 x 7 table of T_d per level is built on the device (49 offsets; 40 are used).
//
// A warp takes 16 targets of one child position c (the c-th children of 16 consecutive parents);
// for each of c's 27 offsets it contracts the real form [Tr -Ti; Ti Tr] (2(p+1) x 2(p+1), padded
// to 8 x 4 DMMA tiles) with the 16 sources' real-ified multipoles on mma.sync.m8n8k4.f64; the
// four warps of a block share the operator, staged once per offset in shared memory.  Sources
// outside the root contribute nothing; empty cells have zero multipoles.  The epilogue adds the
// L2L part from the parent (App. B.5) and writes b_0..b_p of the targets with targets of this
// rank.  The Pascal-form kernel (passes.cu k_down_mma) stays the default; this one runs with
// FMM_M2L_DENSE=1 (quadtree only) -- DESIGN.md §8f has the measured comparison.
#include <stdlib.h>

#include "fmm_internal.cuh"
#include "geometry.cuh"

namespace {

constexpr int BS = 2 * FMM_MAX_P + 2;  // binomial table stride (capi.cu host_binom)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int P>
struct Dense {
  static constexpr int P1 = P + 1;
  static constexpr int MT = (2 * P1 + 7) / 8, KT = (2 * P1 + 3) / 4;
  static constexpr int FRAG = MT * KT * 32;  // doubles of one operator in A-fragment order
  static constexpr int NW = 4;               // warps per block (16 targets each)
};

// operator table of one level: Tfrag[o][mt][kt][lane], o = (dx + 3) * 7 + (dy + 3); A[r][c] at
// lane 4 (r % 8) + (c % 4) of tile (r / 8, c / 4) (m8n8k4 .f64 row-major A fragment)
template <int P>
__global__ void k_dense_ops(double h, int p, const double* __restrict__ binom, double* __restrict__ Tfrag) {
  using D = Dense<P>;
  const int o = blockIdx.x;  // 0..48
  const int dx = o / 7 - 3, dy = o % 7 - 3;
  double* out = Tfrag + (size_t)o * D::FRAG;
  const double zx = h * dx, zy = h * dy;
  const bool used = !(dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1);
  for (int i = threadIdx.x; i < D::FRAG; i += blockDim.x) {
    const int ln = i & 31, kt = (i >> 5) % D::KT, mt = (i >> 5) / D::KT;
    const int r = 8 * mt + (ln >> 2), c = 4 * kt + (ln & 3);
    double v = 0.0;
    if (used && r < 2 * D::P1 && c < 2 * D::P1) {
      const int l = r % D::P1, k = c % D::P1;
      const bool im_row = r >= D::P1, im_col = c >= D::P1;
      if (l <= p && k <= p) {
        // T[l][k] (complex)
        double tr, ti;
        const double d2 = zx * zx + zy * zy;
        const double wr = zx / d2, wi = -zy / d2;  // w = 1 / z0
        if (l == 0 && k == 0) {
          const double mx = -zx, my = __dadd_rn(-zy, 0.0);  // Log(-z0), canonical +0 (D13)
          tr = 0.5 * log(mx * mx + my * my);
          ti = atan2(my, mx);
        } else {
          // w^(l+k) by repeated multiplication (l + k <= 2p)
          double pr = 1.0, pi = 0.0;
          for (int e = 0; e < l + k; ++e) {
            const double nr = pr * wr - pi * wi;
            pi = pr * wi + pi * wr;
            pr = nr;
          }
          double coef;
          if (k == 0) coef = -1.0 / l;
          else coef = ((k & 1) ? -1.0 : 1.0) * (l == 0 ? 1.0 : binom[(l + k - 1) * BS + (k - 1)]);
          tr = coef * pr;
          ti = coef * pi;
        }
        // [yr; yi] = [Tr -Ti; Ti Tr] [ar; ai]
        v = (!im_row && !im_col) ? tr : (!im_row && im_col) ? -ti : (im_row && !im_col) ? ti : tr;
      }
    }
    out[i] = v;
  }
}

template <int P>
__global__ void __launch_bounds__(128) k_m2l_dense(int l, int64_t par0, int64_t npar, int64_t cell0, int64_t cell1,
                                                   int64_t span_l, const int32_t* __restrict__ toff,
                                                   int64_t leaf_lo, int64_t leaf_hi, const double* __restrict__ Tfrag,
                                                   const double2* __restrict__ mp_l, const double2* __restrict__ cen_l,
                                                   const double2* __restrict__ cen_par,
                                                   const double2* __restrict__ loc_par, int p,
                                                   const double* __restrict__ binom, double2* __restrict__ loc_l) {
  using D = Dense<P>;
  constexpr int MT = D::MT, KT = D::KT, P1 = D::P1;
  extern __shared__ double dsm[];
  double* sT = dsm;                                  // two operators (double buffer), A-fragment order
  double* sD = sT + 2 * D::FRAG;                     // per warp: [16 targets][MT * 8] results
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.y;                          // child position of every target of the block
  const int cx = c & 1, cy = c >> 1;
  const int64_t side = (int64_t)1 << l;
  // this lane's B columns: target n = lane / 4 of N tile nt -> parent par0 + 64 bx + 16 w + 8 nt + n
  int64_t tgt[2];
  int ti[2], tj[2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int64_t par = par0 + (int64_t)blockIdx.x * 64 + 16 * w + 8 * nt + (lane >> 2);
    tgt[nt] = par < npar ? 4 * par + c : -1;
    ti[nt] = tgt[nt] >= 0 ? (int)compact2((uint32_t)tgt[nt]) : 0;
    tj[nt] = tgt[nt] >= 0 ? (int)compact2((uint32_t)(tgt[nt] >> 1)) : 0;
  }
  double acc[2][MT][2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[nt][mt][0] = acc[nt][mt][1] = 0.0;
  // the 27 offsets of child position c, in a fixed order
  auto offset_of = [&](int i, int* dx, int* dy) {
    int q = 0;
    for (int dyi = 0; dyi < 6; ++dyi)
      for (int dxi = 0; dxi < 6; ++dxi) {
        const int ddx = dxi - 2 - cx, ddy = dyi - 2 - cy;
        if (ddx >= -1 && ddx <= 1 && ddy >= -1 && ddy <= 1) continue;
        if (q == i) {
          *dx = ddx;
          *dy = ddy;
        }
        ++q;
      }
  };
  // operator staging: cp.async of one operator into one of two shared buffers
  auto stage_op = [&](int i, int buf) {
    int dx, dy;
    offset_of(i, &dx, &dy);
    const double* g = Tfrag + (size_t)((dx + 3) * 7 + (dy + 3)) * D::FRAG;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sT + (size_t)buf * D::FRAG);
    for (int k = threadIdx.x; k < D::FRAG / 2; k += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + 16 * k), "l"(g + 2 * k));
    asm volatile("cp.async.commit_group;");
  };
  // B fragments of offset i: B[k][n] at lane 4n + (k % 4), coefficient k of the real form of a_s
  auto load_b = [&](int i, double (&bf)[KT][2]) {
    int dx, dy;
    offset_of(i, &dx, &dy);
    const double2* src[2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int si = ti[nt] + dx, sj = tj[nt] + dy;
      const bool ok = tgt[nt] >= 0 && si >= 0 && sj >= 0 && si < side && sj < side;
      const int64_t s = ok ? (int64_t)(spread2((uint32_t)si) | (spread2((uint32_t)sj) << 1)) : -1;
      src[nt] = ok ? mp_l + s * (p + 1) : nullptr;
    }
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int k = 4 * kt + (lane & 3);
      const int coef = k < P1 ? k : k - P1;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double v = 0.0;
        if (src[nt] && coef <= p && k < 2 * P1) {
          const double2 a = __ldg(src[nt] + coef);
          v = k < P1 ? a.x : a.y;
        }
        bf[kt][nt] = v;
      }
    }
  };
  double bcur[KT][2], bnext[KT][2];
  stage_op(0, 0);
  load_b(0, bnext);
  for (int i = 0; i < 27; ++i) {
    __syncthreads();  // every warp is done with the buffer operator i + 1 goes to
    if (i + 1 < 27) stage_op(i + 1, (i + 1) & 1);
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) bcur[kt][0] = bnext[kt][0], bcur[kt][1] = bnext[kt][1];
    if (i + 1 < 27) load_b(i + 1, bnext);
    if (i + 1 < 27) asm volatile("cp.async.wait_group 1;");
    else asm volatile("cp.async.wait_group 0;");
    __syncthreads();  // operator i is in shared memory
    const double* sTi = sT + (size_t)(i & 1) * D::FRAG;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double af = sTi[(mt * KT + kt) * 32 + lane];
        dmma884(acc[0][mt][0], acc[0][mt][1], af, bcur[kt][0]);
        dmma884(acc[1][mt][0], acc[1][mt][1], af, bcur[kt][1]);
      }
    }
  }
  // results -> shared memory: C[r][2q + {0,1}] at lane 4r + q, row = 8 mt + lane / 4
  double* myD = sD + (size_t)w * 16 * (MT * 8);
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int r = 8 * mt + (lane >> 2), n0 = 8 * nt + 2 * (lane & 3);
      myD[(size_t)n0 * (MT * 8) + r] = acc[nt][mt][0];
      myD[(size_t)(n0 + 1) * (MT * 8) + r] = acc[nt][mt][1];
    }
  __syncwarp();
  // epilogue per target: L2L from the parent (lane = coefficient) + the M2L sums
  for (int n = 0; n < 16; ++n) {
    const int64_t par = par0 + (int64_t)blockIdx.x * 64 + 16 * w + n;
    if (par >= npar) break;
    const int64_t t = 4 * par + c;
    if (t < cell0 || t >= cell1) continue;
    const int64_t tlo = max(t * span_l, leaf_lo), thi = min((t + 1) * span_l, leaf_hi);
    if (thi <= tlo || toff[thi] == toff[tlo]) continue;  // no targets of this rank below t
    double2 b = make_double2(0.0, 0.0);
    if (l >= 2 && lane <= p) {
      const double2 ct = cen_l[t], cpp = cen_par[par];
      const double2 wv = make_double2(ct.x - cpp.x, ct.y - cpp.y);
      const double2* bp = loc_par + par * (p + 1);
      for (int k = p; k >= lane; --k) {
        const double2 bk = bp[k];
        const double bc = binom[k * BS + lane];
        b = make_double2(b.x * wv.x - b.y * wv.y + bc * bk.x, b.x * wv.y + b.y * wv.x + bc * bk.y);
      }
    }
    if (lane <= p) {
      const double* dn = myD + (size_t)n * (MT * 8);
      loc_l[t * (p + 1) + lane] = make_double2(b.x + dn[lane], b.y + dn[P1 + lane]);
    }
  }
}

}  // namespace

template <int P>
static int launch_dense(fmm_tree_s* t, int l, int64_t c0, int64_t c1, double* Tfrag) {
  using D = Dense<P>;
  const Geo& G = t->g;
  const int p = G.p;
  const double h = ldexp(G.root_size, -l);
  k_dense_ops<P><<<49, 256, 0, t->stream>>>(h, p, t->binom, Tfrag);
  const int64_t par0 = c0 / 4, par1 = (c1 + 3) / 4;
  const size_t smem = sizeof(double) * (2 * D::FRAG + (size_t)D::NW * 16 * D::MT * 8);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_m2l_dense<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)((par1 - par0 + 63) / 64), 4);
  k_m2l_dense<P><<<grid, 128, smem, t->stream>>>(
      l, par0, par1, c0, c1, G.ncells[G.L - l], t->toff, t->leaf_lo, t->leaf_hi, Tfrag, t->mp + G.lvl_off[l] * (p + 1),
      t->centre + G.lvl_off[l], t->centre + G.lvl_off[l - 1], t->loc + G.lvl_off[l - 1] * (p + 1), p, t->binom,
      t->loc + G.lvl_off[l] * (p + 1));
  t->launches += 2;
  return FMM_OK;
}

// levels >= lmin of a quadtree through the dense operators (NEXT-3); returns the first level it
// did not handle (L + 1 when it handled all), so that the caller runs the Pascal form below it.
// Enabled by FMM_M2L_DENSE=1 (FMM_M2L_DENSE_LMIN: first dense level, default L - 1: the coarse
// levels hold too few cells to fill the GPU with 16-target warps and stay on the Pascal form).
bool fmm_m2l_dense_enabled(const fmm_tree_s* t) {
  static const bool on = getenv("FMM_M2L_DENSE") && getenv("FMM_M2L_DENSE")[0] == '1';
  return on && t->g.tiling == FMM_QUADTREE;
}

int fmm_m2l_dense_lmin(int L) {
  const char* s = getenv("FMM_M2L_DENSE_LMIN");
  const int v = s ? atoi(s) : L - 1;
  return v < 2 ? 2 : v;
}

int fmm_m2l_dense_level(fmm_tree_s* t, int l, int64_t c0, int64_t c1, double* Tfrag) {
  const int p = t->g.p;
  if (p <= 8) return launch_dense<8>(t, l, c0, c1, Tfrag);
  if (p <= 12) return launch_dense<12>(t, l, c0, c1, Tfrag);
  if (p <= 16) return launch_dense<16>(t, l, c0, c1, Tfrag);
  if (p <= 20) return launch_dense<20>(t, l, c0, c1, Tfrag);
  if (p <= 24) return launch_dense<24>(t, l, c0, c1, Tfrag);
  if (p <= 28) return launch_dense<28>(t, l, c0, c1, Tfrag);
  return launch_dense<32>(t, l, c0, c1, Tfrag);
}

size_t fmm_m2l_dense_table_bytes(int p) {
  const int P = p <= 8 ? 8 : p <= 12 ? 12 : p <= 16 ? 16 : p <= 20 ? 20 : p <= 24 ? 24 : p <= 28 ? 28 : 32;
  const int P1 = P + 1, MT = (2 * P1 + 7) / 8, KT = (2 * P1 + 3) / 4;
  return sizeof(double) * 49 * (size_t)MT * KT * 32;
}
