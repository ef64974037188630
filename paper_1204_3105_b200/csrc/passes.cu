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

// ------------------------------------------------------------------ P2M (one warp per leaf)
template <int P>
__global__ void __launch_bounds__(128) k_p2m(const double2* __restrict__ sxy, const double* __restrict__ su,
                                             const int32_t* __restrict__ soff, const double2* __restrict__ cen,
                                             int64_t K, int p, double2* __restrict__ mp) {
  int64_t leaf = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= K) return;
  int s0 = soff[leaf], s1 = soff[leaf + 1];
  double2 c = cen[leaf];
  double Sr[P + 1], Si[P + 1];
#pragma unroll
  for (int k = 0; k <= P; ++k) Sr[k] = Si[k] = 0.0;
  for (int i = s0 + lane; i < s1; i += 32) {
    double2 x = sxy[i];
    double u = su[i];
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
  }
#pragma unroll
  for (int k = 0; k <= P; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Sr[k] += __shfl_xor_sync(0xffffffffu, Sr[k], o);
      Si[k] += __shfl_xor_sync(0xffffffffu, Si[k], o);
    }
  }
  double2* out = mp + leaf * (p + 1);
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    if (k <= p && lane == (k & 31)) {
      out[k] = (k == 0) ? make_double2(Sr[0], 0.0) : make_double2(-Sr[k] / k, -Si[k] / k);
    }
  }
}

// ------------------------------------------------------------------ M2M (one warp per parent, lane = coefficient)
__global__ void __launch_bounds__(128) k_m2m(int B, int64_t nparents, int64_t span_l, const int32_t* __restrict__ soff,
                                             const double2* __restrict__ cen_par, const double2* __restrict__ cen_ch,
                                             const double2* __restrict__ mp_ch, int p, const double* __restrict__ binom,
                                             double2* __restrict__ mp_par) {
  int64_t P = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (P >= nparents) return;
  double2 cp = cen_par[P];
  for (int k = lane; k <= p; k += 32) {
    double2 acc = make_double2(0.0, 0.0);
    for (int ch = 0; ch < B; ++ch) {
      int64_t c = P * B + ch;
      if (soff[(c + 1) * span_l] == soff[c * span_l]) continue;
      const double2* a = mp_ch + c * (p + 1);
      double Q = a[0].x;
      if (k == 0) {
        acc.x += Q;
        continue;
      }
      double2 cc = cen_ch[c];
      double2 z0 = make_double2(cc.x - cp.x, cc.y - cp.y);
      double2 h = make_double2(-Q / k, 0.0);
      for (int j = 1; j <= k; ++j) h = cadd(cmul(h, z0), cscale(binom[(k - 1) * BS + (j - 1)], a[j]));
      acc = cadd(acc, h);
    }
    mp_par[P * (p + 1) + k] = acc;
  }
}

// ------------------------------------------------------------------ downward: L2L + M2L (one warp per target cell)
__global__ void __launch_bounds__(128) k_down(int l, int B, int64_t ncells, int64_t span_l,
                                              const int32_t* __restrict__ toff, int64_t leaf_lo, int64_t leaf_hi,
                                              const double2* __restrict__ cen_l, const double2* __restrict__ cen_par,
                                              const double2* __restrict__ loc_par, const int32_t* __restrict__ cand,
                                              const int32_t* __restrict__ ncand,
                                              const unsigned long long* __restrict__ e4mask,
                                              const double2* __restrict__ mp_l, int p,
                                              const double* __restrict__ binom, double2* __restrict__ loc_l) {
  __shared__ double2 at_s[4][32];
  int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 3;
  if (t >= ncells) return;
  int64_t tl = max(t * span_l, leaf_lo), th = min((t + 1) * span_l, leaf_hi);
  if (th <= tl || toff[th] == toff[tl]) return;  // no targets of this rank below t
  double2 ct = cen_l[t];
  double2 acc = make_double2(0.0, 0.0);
  const int L_ = lane;  // output coefficient handled by this lane (p <= 31)
  if (l >= 2) {
    int64_t par = t / B;
    double2 cpp = cen_par[par];
    double2 wv = make_double2(ct.x - cpp.x, ct.y - cpp.y);
    const double2* bp = loc_par + par * (p + 1);
    for (int k = p; k >= 0; --k) {
      double2 bk = bp[k];
      if (k >= L_ && L_ <= p) acc = cadd(cmul(acc, wv), cscale(binom[k * BS + L_], bk));
    }
  }
  int64_t par = t / B;
  unsigned long long mask = e4mask[t];
  const int32_t* cd = cand + par * FMM_CAND_MAX;
  while (mask) {
    int i = __ffsll((long long)mask) - 1;
    mask &= mask - 1;
    int64_t s = cd[i];
    double2 cs = cen_l[s];
    double2 z0 = make_double2(cs.x - ct.x, cs.y - ct.y);
    double2 wv = cinv(z0);
    // w^lane by an inclusive product scan (lane 0 holds 1)
    double2 pw = lane == 0 ? make_double2(1.0, 0.0) : wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double2 y = make_double2(__shfl_up_sync(0xffffffffu, pw.x, o), __shfl_up_sync(0xffffffffu, pw.y, o));
      if (lane >= o) pw = cmul(pw, y);
    }
    const double2* a = mp_l + s * (p + 1);
    double2 ak = (lane <= p) ? a[lane] : make_double2(0.0, 0.0);
    double Q = __shfl_sync(0xffffffffu, ak.x, 0);
    double2 at = cmul(ak, pw);
    if (lane & 1) at = make_double2(-at.x, -at.y);
    at_s[w][lane] = at;
    __syncwarp();
    double2 sum = make_double2(0.0, 0.0);
    if (L_ <= p) {
      for (int k = 1; k <= p; ++k) sum = cadd(sum, cscale(binom[(L_ + k - 1) * BS + (k - 1)], at_s[w][k]));
      if (L_ == 0) {
        double2 lg = clog_principal(ct.x - cs.x, ct.y - cs.y);  // Log(c_L - c_M), D13 (iii)
        acc = cadd(acc, cadd(cscale(Q, lg), sum));
      } else {
        acc = cadd(acc, cmul(pw, make_double2(sum.x - Q / L_, sum.y)));
      }
    }
    __syncwarp();
  }
  if (L_ <= p) loc_l[t * (p + 1) + L_] = acc;
}

// ------------------------------------------------------------------ P2P task list
__global__ void k_chunk_counts(const int32_t* __restrict__ toff, int64_t leaf_lo, int64_t leaf_hi,
                               int32_t* __restrict__ cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t n = leaf_hi - leaf_lo;
  if (i > n) return;
  if (i == n) {
    cnt[i] = 0;
    return;
  }
  int64_t t = leaf_lo + i;
  int nt = toff[t + 1] - toff[t];
  cnt[i] = (nt + 31) / 32;
}
__global__ void k_fill_tasks(const int32_t* __restrict__ toff, int64_t leaf_lo, int64_t leaf_hi,
                             const int32_t* __restrict__ start, int32_t* __restrict__ task_leaf,
                             int32_t* __restrict__ task_start, int32_t* ntask) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t n = leaf_hi - leaf_lo;
  if (i >= n) return;
  int64_t t = leaf_lo + i;
  int nt = toff[t + 1] - toff[t];
  int c = (nt + 31) / 32, s = start[i];
  for (int k = 0; k < c; ++k) {
    task_leaf[s + k] = (int32_t)t;
    task_start[s + k] = toff[t] + 32 * k;
  }
  if (i == n - 1) *ntask = s + c;
}

// ------------------------------------------------------------------ L2P + P2P (one warp per 32-target chunk)
// Sources of each near leaf are staged 32 at a time in shared memory (one coalesced load
// per lane) and read back as broadcasts; log|z|^2 and Arg z come from p2p_math.cuh.
// Tasks are claimed dynamically (one atomic per warp task) for load balance.
__global__ void __launch_bounds__(128) k_p2p_fast(
    const int32_t* __restrict__ task_leaf, const int32_t* __restrict__ task_start, const int32_t* __restrict__ ntask_p,
    int32_t* __restrict__ next_task, const int32_t* __restrict__ toff, const int32_t* __restrict__ soff,
    const double2* __restrict__ txy, const double2* __restrict__ sxy, const double* __restrict__ su,
    const int32_t* __restrict__ near, const int32_t* __restrict__ nnear, const double2* __restrict__ cen_leaf,
    const double2* __restrict__ loc_leaf, int p, int self_mode, const int32_t* __restrict__ tperm,
    const double* __restrict__ tabs, double2* __restrict__ phi, DevStatus* st) {
  __shared__ double2 s_log[P2P_LOG_N];
  __shared__ double2 s_atan[8 * (P2P_ATAN_K + 1)];
  __shared__ double2 s_xy[4][32];
  __shared__ double s_u[4][32];
  p2p_load_tables(tabs, s_log, s_atan);
  const uint32_t a_log = (uint32_t)__cvta_generic_to_shared(s_log);
  const uint32_t a_atan = (uint32_t)__cvta_generic_to_shared(s_atan);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ntask = *ntask_p;
  while (true) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= ntask) break;
    const int t = task_leaf[task];
    const int tpos0 = task_start[task];
    const int nt = min(32, toff[t + 1] - tpos0);
    const int tpos = tpos0 + lane;
    const bool active = lane < nt;
    const double2 y = active ? txy[tpos] : make_double2(1.0e5, 1.0e5);
    double re = 0.0, re_k = 0.0, im = 0.0;
    const int nn = nnear[t];
    for (int qn = 0; qn < nn; ++qn) {
      const int sl = near[(int64_t)t * FMM_NEAR_MAX + qn];
      const int s0 = soff[sl], s1 = soff[sl + 1];
      for (int j0 = s0; j0 < s1; j0 += 32) {
        const int j = j0 + lane;
        if (j < s1) {
          s_xy[w][lane] = sxy[j];
          s_u[w][lane] = su[j];
        }
        __syncwarp();
        const int cnt = min(32, s1 - j0);
        const int excl = (self_mode && sl == t) ? (tpos - j0) : -1;
#pragma unroll 2
        for (int k = 0; k < cnt; ++k) {
          const double2 x = s_xy[w][k];
          const double uu = s_u[w][k];
          double dx = y.x - x.x, dy = y.y - x.y;
          // the pair (i, i) in self mode (D16): dx = dy = 0 exactly; z := 1 + 0i gives
          // log|z|^2 = 0 and Arg z = 0 exactly, so the pair contributes nothing
          if (k == excl) dx = 1.0;
          const double r2 = fma(dx, dx, dy * dy);
          double kd, lz, ag;
          if (__double2hiint(r2) < P2P_SLOW_HI) {  // |z| < 1e-30 (incl. coincident): exact slow path
            kd = 0.0;
            if (r2 == 0.0) {
              if (active) atomicMin(&st->coincident_bad, (unsigned long long)tperm[tpos]);
              lz = 0.0;
              ag = 0.0;
            } else {
              lz = 2.0 * log(hypot(dx, dy));
              ag = atan2(__dadd_rn(dy, 0.0), dx);
            }
          } else {
            p2p_log_split(r2, a_log, &kd, &lz);
            ag = p2p_atan2(dy, dx, a_atan);
          }
          re_k = fma(uu, kd, re_k);  // sum u k  (times ln 2 at the end)
          re = fma(uu, lz, re);
          im = fma(uu, ag, im);
        }
        __syncwarp();
      }
    }
    if (active) {
      const double2 c = cen_leaf[t];
      const double2 z = make_double2(y.x - c.x, y.y - c.y);
      const double2* b = loc_leaf + (int64_t)t * (p + 1);
      double2 acc = b[p];
      for (int k = p - 1; k >= 0; --k) acc = cadd(cmul(acc, z), b[k]);
      re = fma(re_k, P2P_C[10], re) + re_k * P2P_C[11];  // + ln 2 * sum u k
      phi[tperm[tpos]] = make_double2(acc.x + 0.5 * re, acc.y + im);
    }
  }
}

// debug hook: the P2P math on explicit (dx, dy) pairs -> (log |z|^2, Arg z)
__global__ void k_debug_p2p_math(const double2* __restrict__ d, int64_t n, const double* __restrict__ tabs,
                                 double2* __restrict__ out) {
  __shared__ double2 s_log[P2P_LOG_N];
  __shared__ double2 s_atan[8 * (P2P_ATAN_K + 1)];
  p2p_load_tables(tabs, s_log, s_atan);
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double dx = d[i].x, dy = d[i].y;
  double r2 = fma(dx, dx, dy * dy);
  out[i] = make_double2(p2p_log(r2, (uint32_t)__cvta_generic_to_shared(s_log)),
                        p2p_atan2(dy, dx, (uint32_t)__cvta_generic_to_shared(s_atan)));
}

__global__ void __launch_bounds__(128) k_p2p(const int32_t* __restrict__ task_leaf, const int32_t* __restrict__ task_start,
                                             const int32_t* __restrict__ ntask_p, const int32_t* __restrict__ toff,
                                             const int32_t* __restrict__ soff, const double2* __restrict__ txy,
                                             const double2* __restrict__ sxy, const double* __restrict__ su,
                                             const int32_t* __restrict__ near, const int32_t* __restrict__ nnear,
                                             const double2* __restrict__ cen_leaf, const double2* __restrict__ loc_leaf,
                                             int p, int self_mode, const int32_t* __restrict__ tperm,
                                             double2* __restrict__ phi, DevStatus* st) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int ntask = *ntask_p;
  for (int64_t task = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; task < ntask; task += nwarps) {
    int t = task_leaf[task];
    int tpos0 = task_start[task];
    int nt = min(32, toff[t + 1] - tpos0);
    int tpos = tpos0 + lane;
    bool active = lane < nt;
    double2 y = active ? txy[tpos] : make_double2(0.0, 0.0);
    double re = 0.0, im = 0.0;
    int nn = nnear[t];
    for (int q = 0; q < nn; ++q) {
      int sl = near[(int64_t)t * FMM_NEAR_MAX + q];
      int s0 = soff[sl], s1 = soff[sl + 1];
      for (int j0 = s0; j0 < s1; j0 += 32) {
        int j = j0 + lane;
        double2 xs = j < s1 ? sxy[j] : make_double2(0.0, 0.0);
        double us = j < s1 ? su[j] : 0.0;
        int cnt = min(32, s1 - j0);
        for (int k = 0; k < cnt; ++k) {
          double xx = __shfl_sync(0xffffffffu, xs.x, k);
          double xy = __shfl_sync(0xffffffffu, xs.y, k);
          double uu = __shfl_sync(0xffffffffu, us, k);
          double dx = y.x - xx, dy = __dadd_rn(y.y - xy, 0.0);
          bool skip = !active || (self_mode && j0 + k == tpos);
          double r2 = dx * dx + dy * dy;
          if (!skip && r2 == 0.0) {
            atomicMin(&st->coincident_bad, (unsigned long long)tperm[tpos]);
            skip = true;
          }
          if (skip) {
            dx = 1.0;
            dy = 0.0;
            r2 = 1.0;
            uu = 0.0;
          }
          re += uu * log(r2);
          im += uu * atan2(dy, dx);
        }
      }
    }
    if (active) {
      // L2P by Horner at y - c_leaf
      double2 c = cen_leaf[t];
      double2 z = make_double2(y.x - c.x, y.y - c.y);
      const double2* b = loc_leaf + (int64_t)t * (p + 1);
      double2 acc = b[p];
      for (int k = p - 1; k >= 0; --k) acc = cadd(cmul(acc, z), b[k]);
      phi[tperm[tpos]] = make_double2(acc.x + 0.5 * re, acc.y + im);
    }
  }
}

template <int P>
void launch_p2m(fmm_tree_s* t) {
  const Geo& G = t->g;
  int64_t warps = G.K;
  k_p2m<P><<<(unsigned)((warps * 32 + 127) / 128), 128, 0, t->stream>>>(
      t->sxy, t->su, t->soff, t->centre + G.lvl_off[G.L], G.K, G.p, t->mp + G.lvl_off[G.L] * (G.p + 1));
}

}  // namespace

int fmm_stage_upward(fmm_tree_s* t) {
  const Geo& G = t->g;
  cudaStream_t s = t->stream;
  int p = G.p;
  if (p <= 8) launch_p2m<8>(t);
  else if (p <= 12) launch_p2m<12>(t);
  else if (p <= 16) launch_p2m<16>(t);
  else if (p <= 20) launch_p2m<20>(t);
  else if (p <= 24) launch_p2m<24>(t);
  else if (p <= 28) launch_p2m<28>(t);
  else launch_p2m<32>(t);
  t->launches++;
  for (int l = G.L - 1; l >= 1; --l) {
    int64_t np = G.ncells[l];
    k_m2m<<<(unsigned)((np * 32 + 127) / 128), 128, 0, s>>>(
        G.B, np, G.ncells[G.L - l - 1] /* B^(L-l-1) */, t->soff, t->centre + G.lvl_off[l],
        t->centre + G.lvl_off[l + 1], t->mp + G.lvl_off[l + 1] * (p + 1), p, t->binom, t->mp + G.lvl_off[l] * (p + 1));
    t->launches++;
  }
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_stage_downward(fmm_tree_s* t) {
  const Geo& G = t->g;
  cudaStream_t s = t->stream;
  int p = G.p;
  for (int l = 1; l <= G.L; ++l) {
    int64_t nc = G.ncells[l];
    const double2* cen_par = t->centre + G.lvl_off[l - 1];
    const double2* loc_par = t->loc + G.lvl_off[l - 1] * (p + 1);
    k_down<<<(unsigned)((nc * 32 + 127) / 128), 128, 0, s>>>(
        l, G.B, nc, G.ncells[G.L - l] /* B^(L-l) */, t->toff, t->leaf_lo, t->leaf_hi, t->centre + G.lvl_off[l],
        cen_par, loc_par, t->cand + G.lvl_off[l - 1] * FMM_CAND_MAX, t->ncand + G.lvl_off[l - 1],
        t->e4mask + G.lvl_off[l], t->mp + G.lvl_off[l] * (p + 1), p, t->binom, t->loc + G.lvl_off[l] * (p + 1));
    t->launches++;
  }
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_build_tasks(fmm_tree_s* t) {
  cudaStream_t s = t->stream;
  int64_t nl = t->leaf_hi - t->leaf_lo;
  FMM_CUDA_TRY(cudaMemsetAsync(t->ntask, 0, sizeof(int32_t), s));
  if (nl <= 0) return FMM_OK;
  int32_t* cnt = nullptr;
  size_t sb = fmm_scan_scratch_bytes(nl + 1);
  FMM_CUDA_TRY(cudaMallocAsync(&cnt, sizeof(int32_t) * (nl + 1) + sb, s));
  k_chunk_counts<<<(unsigned)((nl + 1 + 255) / 256), 256, 0, s>>>(t->toff, t->leaf_lo, t->leaf_hi, cnt);
  int e = fmm_device_scan_i32(cnt, cnt, nl + 1, cnt + nl + 1, sb, s, &t->launches);
  if (!e) {
    k_fill_tasks<<<(unsigned)((nl + 255) / 256), 256, 0, s>>>(t->toff, t->leaf_lo, t->leaf_hi, cnt, t->task_leaf,
                                                              t->task_start, t->ntask);
  }
  t->launches += 2;
  cudaFreeAsync(cnt, s);
  FMM_CUDA_TRY(cudaGetLastError());
  return e;
}

int fmm_stage_p2p(fmm_tree_s* t, double2* phi) {
  const Geo& G = t->g;
  cudaStream_t s = t->stream;
  static const bool use_ref = getenv("FMM_P2P_LIBDEVICE") && getenv("FMM_P2P_LIBDEVICE")[0] == '1';
  if (use_ref) {  // A/B reference: libdevice log / atan2 (not the product path)
    int blocks = 148 * 32;
    k_p2p<<<blocks, 128, 0, s>>>(t->task_leaf, t->task_start, t->ntask, t->toff, t->soff, t->txy, t->sxy, t->su,
                                 t->near, t->nnear, t->centre + G.lvl_off[G.L],
                                 t->loc + G.lvl_off[G.L] * (G.p + 1), G.p, G.self_mode, t->tperm, phi, t->status);
  } else {
    FMM_CUDA_TRY(cudaMemsetAsync(t->next_task, 0, sizeof(int32_t), s));
    int blocks = 148 * 8;  // persistent-style grid, tasks claimed dynamically
    k_p2p_fast<<<blocks, 128, 0, s>>>(t->task_leaf, t->task_start, t->ntask, t->next_task, t->toff, t->soff, t->txy,
                                      t->sxy, t->su, t->near, t->nnear, t->centre + G.lvl_off[G.L],
                                      t->loc + G.lvl_off[G.L] * (G.p + 1), G.p, G.self_mode, t->tperm, t->p2p_tab,
                                      phi, t->status);
  }
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_debug_p2p_math_launch(const double* dxdy, int64_t n, const double* tabs, double* out, cudaStream_t s) {
  k_debug_p2p_math<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((const double2*)dxdy, n, tabs, (double2*)out);
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}
