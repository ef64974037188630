// capi.cu -- the C ABI of include/fmm_b200.h: configuration checks, device memory
// (one stream-ordered slab per tree), host<->device staging, stage sequencing, exports.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "fmm_internal.cuh"
#include "p2p_math.cuh"

static thread_local std::string g_last_msg;
void fmm_set_error_message(const std::string& s) { g_last_msg = s; }

namespace {

constexpr int BS = 2 * FMM_MAX_P + 2;

std::vector<double> host_binom() {
  std::vector<double> b((size_t)BS * BS, 0.0);
  for (int n = 0; n < BS; ++n) {
    b[(size_t)n * BS] = 1.0;
    for (int k = 1; k <= n; ++k) b[(size_t)n * BS + k] = b[(size_t)(n - 1) * BS + k - 1] + (k < n ? b[(size_t)(n - 1) * BS + k] : 0.0);
  }
  return b;
}

}  // namespace

// tables of p2p_math.cuh, computed once in extended precision (x87 long double)
void fmm_host_p2p_tables(double* tab) {
  memset(tab, 0, sizeof(double) * P2P_TAB_DOUBLES);
  // log tables: N intervals centred on the bit patterns of p2p_math.cuh (1.0 is a centre)
  auto log_table = [&](int off, int n, unsigned long long OFF, int shift) {
    for (int i = 0; i < n; ++i) {
      uint64_t mid = OFF + ((uint64_t)i << shift) + ((uint64_t)1 << (shift - 1));
      double c;
      memcpy(&c, &mid, 8);
      double invc = 1.0 / c;
      tab[off + 2 * i] = invc;
      tab[off + 2 * i + 1] = (double)(-logl((long double)invc));
    }
  };
  log_table(P2P_TAB_LOG, P2P_LOG_N, P2PLogTab<P2P_LOG_N>::OFF, P2PLogTab<P2P_LOG_N>::SHIFT);
  log_table(P2P_TAB_LOGC, P2P_LOGC_N, P2PLogTab<P2P_LOGC_N>::OFF, P2PLogTab<P2P_LOGC_N>::SHIFT);
  const long double PI = acosl(-1.0L);
  // (theta, tau) of octant oct and knot k / K: theta = Arg of the knot direction in the octant,
  // tau = its signed slope tan(theta) (no swap) or -cot(theta) (swap), exactly +-k / K
  auto atan_entry = [&](int oct, int k, int K, double* out) {
    int swap = oct & 1, dxneg = (oct >> 1) & 1, dyneg = (oct >> 2) & 1;
    long double a = atanl((long double)k / K);
    long double t1 = swap ? PI / 2 - a : a;
    long double t2 = dxneg ? PI - t1 : t1;
    long double t3 = dyneg ? -t2 : t2;
    out[0] = (double)t3;
    const double sg = (swap ? -1.0 : 1.0) * ((dxneg ^ dyneg) ? -1.0 : 1.0);
    out[1] = sg * (double)k / K;
  };
  for (int oct = 0; oct < 8; ++oct) {
    for (int k = 0; k < P2P_ATAN_SUB; ++k) atan_entry(oct, k, P2P_ATAN_KS, tab + P2P_TAB_ATAN + 2 * p2p_atan_index(oct, k));
    for (int k = 0; k <= P2P_ATAN_K; ++k) atan_entry(oct, k, P2P_ATAN_K, tab + P2P_TAB_ATANC + 2 * (oct * (P2P_ATAN_K + 1) + k));
  }
}

namespace {

// keep freed tree memory in each device's stream-ordered pool (release threshold = max), once
// per device: trees are built and freed every step, and returning memory to the driver in
// between would make every build pay for fresh allocations
void init_pool_once() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done[dev]) return;
  done[dev] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int64_t ipow64(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

int make_geo(const fmm_config* c, Geo* g) {
  if (!c) return FMM_EBADCFG;
  if (c->tiling < 0 || c->tiling > 2) return FMM_EBADCFG;
  if (c->p < 1 || c->p > FMM_MAX_P - 1) return FMM_EBADCFG;
  if (c->depth < 1 || c->depth > (c->tiling == FMM_SEPTREE ? 10 : 15)) return FMM_EBADCFG;
  if (!(c->root_size > 0.0) || !isfinite(c->root_x) || !isfinite(c->root_y)) return FMM_EBADCFG;
  // the P2P kernel pads with points at |coordinate| 1e30 (p2p.cu): keep the domain far below
  if (!(fabs(c->root_x) + 2.0 * c->root_size < 1e20 && fabs(c->root_y) + 2.0 * c->root_size < 1e20))
    return FMM_EBADCFG;
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) return FMM_EBADCFG;
  // a communicator must describe the same rank / size as the configuration
  if (c->comm && (fmm_comm_nranks(c->comm) != c->nranks || fmm_comm_rank(c->comm) != c->rank)) return FMM_EBADCFG;
  for (int i = 0; i < 5; ++i)
    if (c->reserved[i]) return FMM_EBADCFG;
  if (c->flags & ~FMM_FLAG_TIMING) return FMM_EBADCFG;
  memset(g, 0, sizeof(*g));
  g->tiling = c->tiling;
  g->L = c->depth;
  g->B = c->tiling == FMM_SEPTREE ? 7 : 4;
  g->p = c->p;
  g->self_mode = c->self_mode ? 1 : 0;
  g->K = ipow64(g->B, g->L);
  g->nslot = g->tiling == FMM_QUADTREE ? 9 : (g->tiling == FMM_SEPTREE ? 7 : 13);
  g->lvl_off[0] = 0;
  for (int l = 0; l <= g->L; ++l) {
    g->ncells[l] = ipow64(g->B, l);
    g->lvl_off[l + 1] = g->lvl_off[l] + g->ncells[l];
  }
  g->total_cells = g->lvl_off[g->L + 1];
  g->root_x = c->root_x;
  g->root_y = c->root_y;
  g->root_size = c->root_size;
  if (g->tiling == FMM_SEPTREE) {
    // leaf circumradius r = R0 / (7^floor(L/2) * (L odd ? sqrt 7 : 1))  (reading D8); fixed IEEE sequence
    volatile double den = (double)ipow64(7, g->L / 2);
    if (g->L % 2) den = den * sqrt(7.0);
    volatile double r = c->root_size / den;
    g->sept_r = r;
    volatile double A = 1.5 * r;
    volatile double s3r = 1.7320508075688772 * r;
    volatile double Bc = 0.5 * s3r;
    volatile double D3r = 3.0 * r;
    g->sept_A = A;
    g->sept_Bc = Bc;
    g->sept_D3r = D3r;
  }
  return FMM_OK;
}

// bump allocator over one cudaMallocAsync slab
struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    T* p = (T*)(base ? base + off : nullptr);
    off += bytes;
    return p;
  }
};

void carve(fmm_tree_s* t, Arena& a) {
  const Geo& G = t->g;
  int64_t n = t->n, m = t->m, K = G.K;
  int64_t inner = G.total_cells - G.ncells[G.L];
  t->skey = a.take<uint32_t>(n + 1);
  t->sperm = a.take<int32_t>(n + 1);
  t->soff = a.take<int32_t>(K + 2);
  t->sxy = a.take<double2>(n + 1);
  t->su = a.take<double>(n + 1);
  if (G.self_mode) {
    t->tkey = t->skey;
    t->tperm = t->sperm;
    t->toff = t->soff;
    t->txy = t->sxy;
  } else {
    t->tkey = a.take<uint32_t>(m + 1);
    t->tperm = a.take<int32_t>(m + 1);
    t->toff = a.take<int32_t>(K + 2);
    t->txy = a.take<double2>(m + 1);
  }
  // global leaf CSR: its own arrays only on a multi-rank tree (the local sort keeps a subset)
  if (t->cfg.nranks > 1) {
    t->gsoff = a.take<int32_t>(K + 2);
    t->gtoff = G.self_mode ? t->gsoff : a.take<int32_t>(K + 2);
    t->lflag = a.take<int32_t>(K + 1);
  } else {
    t->gsoff = t->soff;
    t->gtoff = t->toff;
    t->lflag = nullptr;
  }
  t->centre = a.take<double2>(G.total_cells);
  t->cand = a.take<int32_t>(inner * FMM_CAND_MAX);
  t->ncand = a.take<int32_t>(inner);
  t->e4mask = a.take<unsigned long long>(G.total_cells);
  t->near = a.take<int32_t>(K * FMM_NEAR_MAX);
  t->nnear = a.take<int32_t>(K);
  // every (leaf, near leaf) block gives at most ceil(rows / 8) tasks
  t->ntask_cap = (int64_t)G.nslot * (m / 8 + G.K) + 1;
  t->tasks = a.take<int4>(2 * t->ntask_cap);  // two int4 per task (p2p.cu leaf_tasks)
  t->part = a.take<double2>((m + 1) * (int64_t)fmm_part_slots(G));
  t->pskip = a.take<int32_t>(K);
  t->ntask = a.take<int32_t>(1);
  t->next_task = a.take<int32_t>(1);
  t->p2p_tab = a.take<double>(P2P_TAB_DOUBLES);
  t->mp = a.take<double2>(G.total_cells * (G.p + 1));
  t->loc = a.take<double2>(G.total_cells * (G.p + 1));
  t->binom = a.take<double>((size_t)BS * BS);
  t->afr = a.take<double>(FMM_AFR_MAX);
  t->status = a.take<DevStatus>(1);
}


// device buffers of a tree, freed stream-ordered on its stream (the handle stays valid)
void release_buffers(fmm_tree_s* t) {
  cudaStream_t s = t->stream;
  if (t->scratch) cudaFreeAsync(t->scratch, s);
  t->scratch = nullptr;
  t->scratch_bytes = 0;
  for (int i = 0; i < 3; ++i) {
    if (t->staging[i]) cudaFreeAsync(t->staging[i], s);
    t->staging[i] = nullptr;
  }
  if (t->slab) cudaFreeAsync(t->slab, s);
  t->slab = nullptr;
  t->released = 1;
}

int free_tree(fmm_tree_s* t) {
  if (!t) return FMM_OK;
  release_buffers(t);
  for (int i = 0; i < 10; ++i)
    if (t->ev[i]) cudaEventDestroy(t->ev[i]);
  for (int i = 0; i < 2; ++i)
    if (t->xev[i]) cudaEventDestroy(t->xev[i]);
  if (t->xstream) cudaStreamDestroy(t->xstream);
  delete t;
  return FMM_OK;
}

// FMM_DEBUG_SYNC=1: synchronise after every stage and name the stage of a CUDA fault
int debug_sync(cudaStream_t s, const char* stage) {
  static const bool on = getenv("FMM_DEBUG_SYNC") && getenv("FMM_DEBUG_SYNC")[0] == '1';
  if (!on) return FMM_OK;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    fmm_set_error_message(std::string("stage ") + stage + ": " + cudaGetErrorString(e));
    return FMM_ECUDA;
  }
  return FMM_OK;
}

int stage_input(fmm_tree_s* t, const double* src, size_t bytes, int slot, const double** out) {
  if (bytes == 0 || src == nullptr) {
    *out = src;
    return FMM_OK;
  }
  if (is_device_ptr(src)) {
    *out = src;
    return FMM_OK;
  }
  if (t->staging[slot]) cudaFreeAsync(t->staging[slot], t->stream);
  t->staging[slot] = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&t->staging[slot], bytes, t->stream));
  FMM_CUDA_TRY(cudaMemcpyAsync(t->staging[slot], src, bytes, cudaMemcpyHostToDevice, t->stream));
  *out = t->staging[slot];
  return FMM_OK;
}

}  // namespace

extern "C" {

int fmm_version(void) { return 1; }

int fmm_partition(const double* block_work, int64_t nblocks, int64_t leaves_per_block, int64_t K, int32_t rank,
                  int32_t nranks, int64_t* lo, int64_t* hi) {
  if (!lo || !hi || nranks < 1 || rank < 0 || rank >= nranks || nblocks < 0 || leaves_per_block < 1 || K < 0 ||
      (nblocks > 0 && !block_work))
    return FMM_EBADCFG;
  double W = 0.0;
  for (int64_t b = 0; b < nblocks; ++b) W += block_work[b] > 0.0 ? block_work[b] : 0.0;
  // cut(r): the block boundary whose prefix work is closest to r W / nranks (monotone in r)
  auto cut = [&](int32_t r) -> int64_t {
    if (r <= 0) return 0;
    if (r >= nranks) return nblocks;
    double target = W * (double)r / (double)nranks, pre = 0.0;
    int64_t b = 0;
    while (b < nblocks && pre + (block_work[b] > 0.0 ? block_work[b] : 0.0) <= target) {
      pre += block_work[b] > 0.0 ? block_work[b] : 0.0;
      ++b;
    }
    if (b < nblocks) {
      double next = pre + (block_work[b] > 0.0 ? block_work[b] : 0.0);
      if (next - target < target - pre) ++b;
    }
    return b;
  };
  int64_t c0 = cut(rank), c1 = cut(rank + 1);
  *lo = std::min(c0 * leaves_per_block, K);
  *hi = std::min(c1 * leaves_per_block, K);
  return FMM_OK;
}

// ------------------------------------------------------------------ NEXT-2: depth selection
// The appendix cost model or a per-unit device-time model:
//   paper: (M+N) P + K B/(B-1) (P4+2) P^2 + M (P2 s + P)          (s = N / K, K = B^L)
//   unit : c0 + c_point (N+M)(p+1) + c_cell K B/(B-1) (P4+2) (p+1)^2 + c_pair M P2 s + c_leaf K
static void cost_params(int tiling, double* B, double* P4, double* P2) {
  if (tiling == FMM_QUADTREE) {
    *B = 4.0; *P4 = 27.0; *P2 = 9.0;
  } else if (tiling == FMM_SEPTREE) {
    *B = 7.0; *P4 = 42.0; *P2 = 7.0;
  } else {
    *B = 4.0; *P4 = 39.0; *P2 = 13.0;
  }
}

int fmm_predict_cost(int32_t tiling, int64_t n, int64_t m, int32_t p, int32_t depth, const fmm_unit_costs* uc,
                     double* cost) {
  if (tiling < 0 || tiling > 2 || n < 0 || m < 0 || p < 1 || depth < 1 || depth > 20 || !cost) return FMM_EBADCFG;
  double B, P4, P2;
  cost_params(tiling, &B, &P4, &P2);
  const double K = pow(B, depth), N = (double)n, M = (double)m, s = N / K, P = (double)p;
  if (!uc) {
    *cost = (M + N) * P + K * B / (B - 1.0) * (P4 + 2.0) * P * P + M * (P2 * s + P);
  } else {
    const double P1 = P + 1.0;
    *cost = uc->c0 + uc->c_point * (N + M) * P1 + uc->c_cell * K * B / (B - 1.0) * (P4 + 2.0) * P1 * P1 +
            uc->c_pair * M * P2 * s + uc->c_leaf * K;
  }
  return FMM_OK;
}

int fmm_choose_depth(int32_t tiling, int64_t n, int64_t m, int32_t p, const fmm_unit_costs* uc, int32_t* depth) {
  if (!depth) return FMM_EBADCFG;
  const int maxd = tiling == FMM_SEPTREE ? 10 : 15;
  int best = 1;
  double bc = 0.0;
  for (int L = 1; L <= maxd; ++L) {
    double c;
    int e = fmm_predict_cost(tiling, n, m, p, L, uc, &c);
    if (e) return e;
    if (L == 1 || c < bc) {
      bc = c;
      best = L;
    }
  }
  *depth = best;
  return FMM_OK;
}

int fmm_pool_reserve(size_t bytes) {
  init_pool_once();
  void* p = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync(&p, bytes, 0));
  FMM_CUDA_TRY(cudaFreeAsync(p, 0));
  FMM_CUDA_TRY(cudaStreamSynchronize(0));
  return FMM_OK;
}

size_t fmm_tree_bytes(fmm_tree_t t) { return t ? t->slab_bytes : 0; }

const char* fmm_error_string(int code) {
  switch (code) {
    case FMM_OK: return "ok";
    case FMM_EBADCFG: return "invalid configuration or argument";
    case FMM_EDOMAIN: return "point outside the root domain";
    case FMM_ECOINCIDENT: return "target coincides with a source";
    case FMM_ECUDA: return "CUDA error";
    case FMM_ENOMEM: return "device allocation failed";
    case FMM_EEXTENSION: return "unsupported request";
    default: return "unknown error";
  }
}

const char* fmm_last_error_message(void) { return g_last_msg.c_str(); }

int fmm_build_tree(const fmm_config* cfg, const double* src_xy, const double* src_u, int64_t n,
                   const double* tgt_xy, int64_t m, void* stream, fmm_tree_t* out) {
  if (!out) return FMM_EBADCFG;
  *out = nullptr;
  Geo g;
  int e = make_geo(cfg, &g);
  if (e) return e;
  if (n < 0 || m < 0) return FMM_EBADCFG;
  // limits of the build's device scans (leaf counts, task counts, radix digit histograms)
  if (g.K + 2 > fmm_scan_max_entries()) {
    fmm_set_error_message("depth too large for the build: at most 12 (quadtree, triangle) or 9 (septree) levels");
    return FMM_EBADCFG;
  }
  if (n > FMM_MAX_POINTS || m > FMM_MAX_POINTS) {
    fmm_set_error_message("too many points: at most 2^27 sources and 2^27 targets per tree");
    return FMM_EBADCFG;
  }
  if (cfg->self_mode) {
    if (m != n && m != 0 && tgt_xy) return FMM_EBADCFG;
    m = n;
  }
  if ((n > 0 && (!src_xy || !src_u)) || (!cfg->self_mode && m > 0 && !tgt_xy)) return FMM_EBADCFG;
  init_pool_once();
  fmm_tree_s* t = new fmm_tree_s();
  memset((void*)t, 0, sizeof(*t));
  t->cfg = *cfg;
  t->g = g;
  t->stream = (cudaStream_t)stream;
  t->n = n;
  t->m = m;
  t->leaf_lo = 0;  // the rank's range is set by fmm_stage_near_partition
  t->leaf_hi = g.K;
  t->comm = cfg->comm;
  cudaStream_t s = t->stream;
  // inputs
  e = stage_input(t, src_xy, (size_t)n * 16, 0, &t->src_xy_in);
  if (!e) e = stage_input(t, src_u, (size_t)n * 8, 1, &t->src_u_in);
  if (!e && !g.self_mode) e = stage_input(t, tgt_xy, (size_t)m * 16, 2, &t->tgt_xy_in);
  if (e) {
    free_tree(t);
    return e;
  }
  // one slab for every tree buffer
  Arena sizer;
  carve(t, sizer);
  char* slab = nullptr;
  cudaError_t ce = cudaMallocAsync((void**)&slab, sizer.off, s);
  if (ce != cudaSuccess) {
    fmm_set_error_message(std::string("cudaMallocAsync slab: ") + cudaGetErrorString(ce));
    free_tree(t);
    return ce == cudaErrorMemoryAllocation ? FMM_ENOMEM : FMM_ECUDA;
  }
  Arena a;
  a.base = slab;
  carve(t, a);
  t->slab = slab;
  t->slab_bytes = sizer.off;
  // binomials and P2P tables: one pinned host copy per process, so that these copies stay
  // asynchronous (a pageable source would synchronise the stream with the host)
  static double* hconst = nullptr;
  static cudaError_t hconst_err = cudaSuccess;
  static std::once_flag hconst_once;
  std::call_once(hconst_once, [] {
    const size_t nb = (size_t)BS * BS;
    hconst_err = cudaHostAlloc((void**)&hconst, (nb + P2P_TAB_DOUBLES + 7 * FMM_AFR_MAX) * sizeof(double),
                               cudaHostAllocPortable);
    if (hconst_err != cudaSuccess) return;
    std::vector<double> hb = host_binom();
    memcpy(hconst, hb.data(), nb * sizeof(double));
    fmm_host_p2p_tables(hconst + nb);
    // the downward kernel's A fragments for every template order 8, 12, ..., 32
    for (int i = 0; i < 7; ++i) {
      double* dst = hconst + nb + P2P_TAB_DOUBLES + (size_t)i * FMM_AFR_MAX;
      memset(dst, 0, sizeof(double) * FMM_AFR_MAX);
      fmm_down_afr_fill(8 + 4 * i, hb.data(), dst);
    }
  });
  ce = hconst_err;
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(t->binom, hconst, (size_t)BS * BS * sizeof(double), cudaMemcpyHostToDevice, s);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(t->p2p_tab, hconst + (size_t)BS * BS, P2P_TAB_DOUBLES * sizeof(double),
                         cudaMemcpyHostToDevice, s);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(t->afr,
                         hconst + (size_t)BS * BS + P2P_TAB_DOUBLES + (size_t)((fmm_down_order(g.p) - 8) / 4) * FMM_AFR_MAX,
                         FMM_AFR_MAX * sizeof(double), cudaMemcpyHostToDevice, s);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(t->status, 0xff, sizeof(DevStatus), s);
  if (ce != cudaSuccess) {
    fmm_set_error_message(cudaGetErrorString(ce));
    free_tree(t);
    return FMM_ECUDA;
  }
  if (cfg->flags & FMM_FLAG_TIMING) {
    e = fmm_set_timing(t, 1);
    if (e) {
      free_tree(t);
      return e;
    }
    cudaEventRecord(t->ev[0], s);
  }
  e = fmm_stage_keys_sort(t);
  if (!e) e = debug_sync(s, "keys+sort");
  if (t->timing) cudaEventRecord(t->ev[1], s);
  if (!e) e = fmm_stage_tables_lists(t);
  if (!e) e = debug_sync(s, "tables+lists");
  if (!e) e = fmm_build_tasks(t);
  if (!e) e = debug_sync(s, "tasks");
  if (t->timing) cudaEventRecord(t->ev[2], s);
  t->build_timed = t->timing;
  if (e) {
    free_tree(t);
    return e;
  }
  *out = t;
  return FMM_OK;
}

int fmm_set_strengths(fmm_tree_t t, const double* src_u, void* stream) {
  if (!t || t->released || (t->n > 0 && !src_u)) return FMM_EBADCFG;
  if (stream) t->stream = (cudaStream_t)stream;
  const double* u = nullptr;
  int e = stage_input(t, src_u, (size_t)t->n * 8, 1, &u);
  if (!e) e = fmm_stage_gather_strengths(t, u);
  return e;
}

// the first half of an evaluation: upward pass (own source leaves), the multipole all-reduce
// on the side stream when a communicator is set, and the P2P pair kernel, which needs no
// multipoles and so overlaps the exchange
int fmm_evaluate_begin(fmm_tree_t t, void* stream) {
  if (!t || t->released) return FMM_EBADCFG;
  if (stream) t->stream = (cudaStream_t)stream;
  cudaStream_t s = t->stream;
  t->begun = 0;
  if (t->m == 0) return FMM_OK;
  if (t->timing) cudaEventRecord(t->ev[3], s);
  int e = fmm_stage_upward(t);
  if (!e) e = debug_sync(s, "upward");
  if (t->timing) cudaEventRecord(t->ev[4], s);
  if (!e && t->comm) {
    if (!t->xstream) {
      int lo = 0, hi = 0;
      FMM_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      FMM_CUDA_TRY(cudaStreamCreateWithPriority(&t->xstream, cudaStreamNonBlocking, hi));
      for (int i = 0; i < 2; ++i) FMM_CUDA_TRY(cudaEventCreateWithFlags(&t->xev[i], cudaEventDisableTiming));
    }
    FMM_CUDA_TRY(cudaEventRecord(t->xev[0], s));
    FMM_CUDA_TRY(cudaStreamWaitEvent(t->xstream, t->xev[0], 0));
    const Geo& G = t->g;
    e = fmm_comm_allreduce_sum_f64(t->comm, (double*)t->mp, (size_t)G.total_cells * (G.p + 1) * 2, t->xstream);
    if (!e) FMM_CUDA_TRY(cudaEventRecord(t->xev[1], t->xstream));
  }
  if (!e) e = fmm_stage_p2p_pairs(t);
  if (!e) e = debug_sync(s, "p2p pairs");
  if (t->timing) cudaEventRecord(t->ev[7], s);
  if (!e) t->begun = 1;
  return e;
}

// the second half: (wait for the exchange) M2L + L2L over every level, near-field sums + L2P
int fmm_evaluate_end(fmm_tree_t t, double* phi_out, void* stream) {
  if (!t || t->released) return FMM_EBADCFG;
  if (stream) t->stream = (cudaStream_t)stream;
  cudaStream_t s = t->stream;
  if (t->m == 0) return FMM_OK;
  if (!phi_out || !t->begun) return FMM_EBADCFG;
  t->begun = 0;
  bool dev = is_device_ptr(phi_out);
  double2* phi = (double2*)phi_out;
  double2* tmp = nullptr;
  if (!dev) {
    FMM_CUDA_TRY(cudaMallocAsync((void**)&tmp, (size_t)t->m * 16, s));
    phi = tmp;
    // other ranks' targets are not written: keep the caller's values for them
    if (t->cfg.nranks > 1)
      FMM_CUDA_TRY(cudaMemcpyAsync(tmp, phi_out, (size_t)t->m * 16, cudaMemcpyHostToDevice, s));
  }
  if (t->comm) FMM_CUDA_TRY(cudaStreamWaitEvent(s, t->xev[1], 0));
  int e = fmm_stage_downward(t);
  if (!e) e = debug_sync(s, "downward");
  if (t->timing) cudaEventRecord(t->ev[5], s);
  if (!e) e = fmm_stage_p2p_finish(t, phi);
  if (!e) e = debug_sync(s, "p2p finish");
  if (t->timing) cudaEventRecord(t->ev[6], s);
  t->eval_timed = t->timing;
  if (!e && !dev) FMM_CUDA_TRY(cudaMemcpyAsync(phi_out, tmp, (size_t)t->m * 16, cudaMemcpyDeviceToHost, s));
  if (tmp) cudaFreeAsync(tmp, s);
  return e;
}

int fmm_evaluate(fmm_tree_t t, double* phi_out, void* stream) {
  if (!t || t->released) return FMM_EBADCFG;
  if (t->m > 0 && !phi_out) return FMM_EBADCFG;
  if (t->cfg.nranks > 1 && !t->comm) {
    fmm_set_error_message("fmm_evaluate: nranks > 1 needs cfg->comm (or fmm_evaluate_begin / _end with the "
                          "multipole exchange done by the caller)");
    return FMM_EBADCFG;
  }
  int e = fmm_evaluate_begin(t, stream);
  if (!e) e = fmm_evaluate_end(t, phi_out, stream);
  return e;
}

int fmm_multipole_buffer(fmm_tree_t t, void** dev_ptr, size_t* bytes) {
  if (!t || t->released) return FMM_EBADCFG;
  if (dev_ptr) *dev_ptr = (void*)t->mp;
  if (bytes) *bytes = (size_t)t->g.total_cells * (t->g.p + 1) * sizeof(double2);
  return FMM_OK;
}

int fmm_status(fmm_tree_t t) {
  if (!t || t->released) return FMM_EBADCFG;
  FMM_CUDA_TRY(cudaStreamSynchronize(t->stream));
  DevStatus st;
  FMM_CUDA_TRY(cudaMemcpy(&st, t->status, sizeof(st), cudaMemcpyDeviceToHost));
  if (st.domain_bad != ~0ull) return FMM_EDOMAIN;
  if (st.coincident_bad != ~0ull) return FMM_ECOINCIDENT;
  return FMM_OK;
}

int64_t fmm_last_error_index(fmm_tree_t t) {
  if (!t || t->released) return -1;
  if (cudaStreamSynchronize(t->stream) != cudaSuccess) return -1;
  DevStatus st;
  if (cudaMemcpy(&st, t->status, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  if (st.domain_bad != ~0ull) return (int64_t)st.domain_bad;
  if (st.coincident_bad != ~0ull) return (int64_t)st.coincident_bad;
  return -1;
}

int fmm_set_timing(fmm_tree_t t, int32_t enable) {
  if (!t) return FMM_EBADCFG;
  if (enable && !t->ev[0])
    for (int i = 0; i < 10; ++i) FMM_CUDA_TRY(cudaEventCreate(&t->ev[i]));
  t->timing = enable;
  return FMM_OK;
}
/* stage times: {keys + sort, lists + tasks, P2P pair kernel, upward, downward (incl. the wait
 * for the multipole exchange), pair kernel + near-field sums / L2P}; the evaluation order is
 * upward (ev3 -> ev4), pairs (ev4 -> ev7), downward (ev7 -> ev5), finish (ev5 -> ev6) */
int fmm_stage_times(fmm_tree_t t, float* ms6) {
  if (!t || !ms6) return FMM_EBADCFG;
  for (int i = 0; i < 6; ++i) ms6[i] = 0.f;
  if (!t->timing) return FMM_OK;
  if (t->build_timed) {
    FMM_CUDA_TRY(cudaEventSynchronize(t->ev[2]));
    cudaEventElapsedTime(&ms6[0], t->ev[0], t->ev[1]);
    cudaEventElapsedTime(&ms6[1], t->ev[1], t->ev[2]);
  }
  if (t->eval_timed) {
    FMM_CUDA_TRY(cudaEventSynchronize(t->ev[6]));
    float fin = 0.f;
    cudaEventElapsedTime(&ms6[2], t->ev[4], t->ev[7]);
    cudaEventElapsedTime(&ms6[3], t->ev[3], t->ev[4]);
    cudaEventElapsedTime(&ms6[4], t->ev[7], t->ev[5]);
    cudaEventElapsedTime(&fin, t->ev[5], t->ev[6]);
    ms6[5] = ms6[2] + fin;
  }
  return FMM_OK;
}

int fmm_build_times(fmm_tree_t t, float* ms4) {
  if (!t || !ms4) return FMM_EBADCFG;
  for (int i = 0; i < 4; ++i) ms4[i] = 0.f;
  if (!t->timing || !t->build_timed) return FMM_OK;
  FMM_CUDA_TRY(cudaEventSynchronize(t->ev[2]));
  cudaEventElapsedTime(&ms4[0], t->ev[0], t->ev[8]);
  cudaEventElapsedTime(&ms4[1], t->ev[8], t->ev[9]);
  cudaEventElapsedTime(&ms4[2], t->ev[9], t->ev[1]);
  cudaEventElapsedTime(&ms4[3], t->ev[1], t->ev[2]);
  return FMM_OK;
}

int fmm_rank_range(fmm_tree_t t, int64_t* lo, int64_t* hi) {
  if (!t) return FMM_EBADCFG;
  if (lo) *lo = t->leaf_lo;
  if (hi) *hi = t->leaf_hi;
  return FMM_OK;
}

int64_t fmm_launch_count(fmm_tree_t t) { return t ? t->launches : -1; }

void fmm_free(fmm_tree_t t) { free_tree(t); }

int fmm_release(fmm_tree_t t) {
  if (!t) return FMM_EBADCFG;
  release_buffers(t);
  return FMM_OK;
}

int fmm_direct(const double* src_xy, const double* src_u, int64_t n, const double* tgt_xy, int64_t m,
               int32_t self_mode, double* phi_out, void* stream) {
  if (n < 0 || m < 0 || (self_mode && m != n)) return FMM_EBADCFG;
  if (m == 0) return FMM_OK;
  if (!phi_out || (n > 0 && (!src_xy || !src_u)) || (!self_mode && !tgt_xy)) return FMM_EBADCFG;
  init_pool_once();
  cudaStream_t s = (cudaStream_t)stream;
  // device copies of host inputs / output, the P2P tables and the error word in one allocation
  const bool dsx = is_device_ptr(src_xy), dsu = is_device_ptr(src_u), dphi = is_device_ptr(phi_out);
  const double* t_in = self_mode ? src_xy : tgt_xy;
  const bool dtx = is_device_ptr(t_in);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t o_sx = dsx ? 0 : take((size_t)n * 16), o_su = dsu ? 0 : take((size_t)n * 8);
  const size_t o_tx = (dtx || self_mode) ? 0 : take((size_t)m * 16), o_phi = dphi ? 0 : take((size_t)m * 16);
  const size_t o_tab = take(P2P_TAB_DOUBLES * 8), o_bad = take(8);
  char* buf = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&buf, off, s));
  const double* sx = dsx ? src_xy : (const double*)(buf + o_sx);
  const double* su = dsu ? src_u : (const double*)(buf + o_su);
  if (!dsx) FMM_CUDA_TRY(cudaMemcpyAsync(buf + o_sx, src_xy, (size_t)n * 16, cudaMemcpyHostToDevice, s));
  if (!dsu) FMM_CUDA_TRY(cudaMemcpyAsync(buf + o_su, src_u, (size_t)n * 8, cudaMemcpyHostToDevice, s));
  const double* tx = self_mode ? sx : (dtx ? tgt_xy : (const double*)(buf + o_tx));
  if (!self_mode && !dtx) FMM_CUDA_TRY(cudaMemcpyAsync(buf + o_tx, tgt_xy, (size_t)m * 16, cudaMemcpyHostToDevice, s));
  double* ph = dphi ? phi_out : (double*)(buf + o_phi);
  std::vector<double> tab(P2P_TAB_DOUBLES);
  fmm_host_p2p_tables(tab.data());
  FMM_CUDA_TRY(cudaMemcpyAsync(buf + o_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s));
  FMM_CUDA_TRY(cudaMemsetAsync(buf + o_bad, 0xff, 8, s));
  int e = fmm_direct_launch(sx, su, n, tx, m, self_mode, (const double*)(buf + o_tab), ph,
                            (unsigned long long*)(buf + o_bad), s);
  unsigned long long bad = ~0ull;
  if (!e && !dphi) FMM_CUDA_TRY(cudaMemcpyAsync(phi_out, ph, (size_t)m * 16, cudaMemcpyDeviceToHost, s));
  if (!e) FMM_CUDA_TRY(cudaMemcpyAsync(&bad, buf + o_bad, 8, cudaMemcpyDeviceToHost, s));
  FMM_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFreeAsync(buf, s);
  if (e) return e;
  if (bad != ~0ull) {
    fmm_set_error_message("coincident source and target at target index " + std::to_string(bad));
    return FMM_ECOINCIDENT;
  }
  return FMM_OK;
}

int fmm_sample_cells(const fmm_config* cfg, const int64_t* cells, int64_t ncells, int32_t per_cell, uint64_t seed,
                     int64_t first, double* xy, double* u, void* stream) {
  Geo g;
  int e = make_geo(cfg, &g);
  if (e) return e;
  if (ncells < 0 || per_cell < 0 || first < 0) return FMM_EBADCFG;
  if (!cells && ncells > g.K) return FMM_EBADCFG;
  if (per_cell > 0 && ncells > (((int64_t)1 << 60) - first) / per_cell) return FMM_EBADCFG;
  const int64_t npts = ncells * (int64_t)per_cell;
  if (npts == 0) return FMM_OK;
  if (!is_device_ptr(xy) || (u && !is_device_ptr(u)) || (cells && !is_device_ptr(cells))) return FMM_EBADCFG;
  // leaf polygon (D22): half-edge a and apothem b of the rectangle, apothem directions
  SamplePoly P;
  if (g.tiling == FMM_QUADTREE) {  // square of side S 2^-L; edges facing 0, pi/2, pi, 3pi/2
    P.nsides = 4, P.step = 3, P.off = 0;
    P.a = 0.5 * ldexp(g.root_size, -g.L);
    P.b = P.a;
  } else if (g.tiling == FMM_SEPTREE) {  // hexagon of circumradius r (D8), a vertex at angle 0
    P.nsides = 6, P.step = 2, P.off = 1;
    P.a = 0.5 * g.sept_r;
    P.b = 0.8660254037844386 * g.sept_r;
  } else {  // triangle of circumradius R0 2^-L; off (1 upright, 3 inverted) per cell
    const double R = ldexp(g.root_size, -g.L);
    P.nsides = 3, P.step = 4, P.off = 1;
    P.a = 0.8660254037844386 * R;
    P.b = 0.5 * R;
  }
  init_pool_once();
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* dbad = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&dbad, 8, s));
  FMM_CUDA_TRY(cudaMemsetAsync(dbad, 0xff, 8, s));
  e = fmm_sample_launch(g, cells, ncells, per_cell, seed, first, P, xy, u, dbad, s);
  unsigned long long bad = ~0ull;
  if (!e) FMM_CUDA_TRY(cudaMemcpyAsync(&bad, dbad, 8, cudaMemcpyDeviceToHost, s));
  FMM_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFreeAsync(dbad, s);
  if (e) return e;
  if (bad != ~0ull) {
    fmm_set_error_message("cell outside [0, B^L) at cells index " + std::to_string(bad));
    return FMM_EDOMAIN;
  }
  return FMM_OK;
}

int fmm_debug_p2p_math(const double* dxdy, int64_t n, double* out, void* stream) {
  if (n <= 0) return FMM_OK;
  if (!is_device_ptr(dxdy) || !is_device_ptr(out)) return FMM_EBADCFG;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double> tab(P2P_TAB_DOUBLES);
  fmm_host_p2p_tables(tab.data());
  double* dtab = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&dtab, tab.size() * 8, s));
  FMM_CUDA_TRY(cudaMemcpyAsync(dtab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s));
  int e = fmm_debug_p2p_math_launch(dxdy, n, dtab, out, s);
  FMM_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFreeAsync(dtab, s);
  return e;
}

static int copy_out(const void* src_dev, size_t bytes, void* host_buf, size_t cap, size_t* needed) {
  if (needed) *needed = bytes;
  if (host_buf && bytes) FMM_CUDA_TRY(cudaMemcpy(host_buf, src_dev, std::min(bytes, cap), cudaMemcpyDeviceToHost));
  return FMM_OK;
}
static int copy_host(const void* src, size_t bytes, void* host_buf, size_t cap, size_t* needed) {
  if (needed) *needed = bytes;
  if (host_buf && bytes) memcpy(host_buf, src, std::min(bytes, cap));
  return FMM_OK;
}

int fmm_export(fmm_tree_t t, int32_t what, int32_t level, void* host_buf, size_t bytes, size_t* needed) {
  if (!t || t->released) return FMM_EBADCFG;
  FMM_CUDA_TRY(cudaStreamSynchronize(t->stream));
  const Geo& G = t->g;
  int64_t K = G.K;
  if ((what == FMM_X_CENTRES || what == FMM_X_E4_OWNERS || what == FMM_X_E4_OFFSETS || what == FMM_X_E4_ENTRIES ||
       what == FMM_X_MULTIPOLE || what == FMM_X_LOCAL) &&
      (level < 0 || level > G.L))
    return FMM_EBADCFG;
  switch (what) {
    case FMM_X_SRC_KEYS: return copy_out(t->skey, (size_t)t->n * 4, host_buf, bytes, needed);
    case FMM_X_TGT_KEYS: return copy_out(t->tkey, (size_t)t->m * 4, host_buf, bytes, needed);
    case FMM_X_SRC_PERM: return copy_out(t->sperm, (size_t)t->n_loc * 4, host_buf, bytes, needed);
    case FMM_X_TGT_PERM: return copy_out(t->tperm, (size_t)t->m_loc * 4, host_buf, bytes, needed);
    case FMM_X_CENTRES:
      return copy_out(t->centre + G.lvl_off[level], (size_t)G.ncells[level] * 16, host_buf, bytes, needed);
    case FMM_X_MULTIPOLE:
      return copy_out(t->mp + G.lvl_off[level] * (G.p + 1), (size_t)G.ncells[level] * (G.p + 1) * 16, host_buf,
                      bytes, needed);
    case FMM_X_LOCAL:
      return copy_out(t->loc + G.lvl_off[level] * (G.p + 1), (size_t)G.ncells[level] * (G.p + 1) * 16, host_buf,
                      bytes, needed);
    default: break;
  }
  // host-side views that need the CSR offsets
  std::vector<int32_t> so(K + 2), to(K + 2);
  FMM_CUDA_TRY(cudaMemcpy(so.data(), t->soff, (K + 2) * 4, cudaMemcpyDeviceToHost));
  FMM_CUDA_TRY(cudaMemcpy(to.data(), t->toff, (K + 2) * 4, cudaMemcpyDeviceToHost));
  if (what == FMM_X_SRC_OFFSETS || what == FMM_X_TGT_OFFSETS) {
    std::vector<int64_t> o(K + 1);
    const std::vector<int32_t>& src = what == FMM_X_SRC_OFFSETS ? so : to;
    for (int64_t i = 0; i <= K; ++i) o[i] = src[i];
    return copy_host(o.data(), o.size() * 8, host_buf, bytes, needed);
  }
  auto tcount = [&](int l, int64_t c) -> int64_t {
    int64_t span = ipow64(G.B, G.L - l);
    int64_t lo = std::max(c * span, t->leaf_lo), hi = std::min((c + 1) * span, t->leaf_hi);
    return hi > lo ? to[hi] - to[lo] : 0;
  };
  std::vector<int32_t> owners, entries;
  std::vector<int64_t> offs(1, 0);
  int64_t m2l_ops = 0, p2p_pairs = 0, ne_src = 0, ne_tgt = 0;
  bool want_near = what == FMM_X_NEAR_OWNERS || what == FMM_X_NEAR_OFFSETS || what == FMM_X_NEAR_ENTRIES;
  bool want_e4 = what == FMM_X_E4_OWNERS || what == FMM_X_E4_OFFSETS || what == FMM_X_E4_ENTRIES;
  if (want_near || what == FMM_X_COUNTERS) {
    std::vector<int32_t> nr(K * FMM_NEAR_MAX), nn(K);
    FMM_CUDA_TRY(cudaMemcpy(nr.data(), t->near, nr.size() * 4, cudaMemcpyDeviceToHost));
    FMM_CUDA_TRY(cudaMemcpy(nn.data(), t->nnear, nn.size() * 4, cudaMemcpyDeviceToHost));
    for (int64_t leaf = 0; leaf < K; ++leaf) ne_src += so[leaf + 1] > so[leaf];
    for (int64_t leaf = t->leaf_lo; leaf < t->leaf_hi; ++leaf) {
      int64_t nt = to[leaf + 1] - to[leaf];
      if (nt == 0) continue;
      ++ne_tgt;
      owners.push_back((int32_t)leaf);
      int64_t ns = 0;
      for (int q = 0; q < nn[leaf]; ++q) {
        int32_t s = nr[leaf * FMM_NEAR_MAX + q];
        entries.push_back(s);
        ns += so[s + 1] - so[s];
      }
      p2p_pairs += nt * ns - (G.self_mode ? nt : 0);
      offs.push_back((int64_t)entries.size());
    }
  }
  if (want_e4 || what == FMM_X_COUNTERS) {
    int l0 = want_e4 ? level : 1, l1 = want_e4 ? level : G.L;
    if (want_e4) {
      owners.clear();
      entries.clear();
      offs.assign(1, 0);
    }
    for (int l = std::max(l0, 1); l <= l1; ++l) {
      int64_t nc = G.ncells[l], np = G.ncells[l - 1];
      std::vector<int32_t> cand(np * FMM_CAND_MAX), ncand(np);
      std::vector<unsigned long long> mask(nc);
      FMM_CUDA_TRY(cudaMemcpy(cand.data(), t->cand + G.lvl_off[l - 1] * FMM_CAND_MAX, cand.size() * 4,
                              cudaMemcpyDeviceToHost));
      FMM_CUDA_TRY(cudaMemcpy(ncand.data(), t->ncand + G.lvl_off[l - 1], np * 4, cudaMemcpyDeviceToHost));
      FMM_CUDA_TRY(cudaMemcpy(mask.data(), t->e4mask + G.lvl_off[l], nc * 8, cudaMemcpyDeviceToHost));
      for (int64_t c = 0; c < nc; ++c) {
        if (tcount(l, c) == 0) continue;
        int64_t P = c / G.B;
        unsigned long long mk = mask[c];
        if (want_e4) owners.push_back((int32_t)c);
        for (int i = 0; i < ncand[P] && i < 64; ++i)
          if (mk >> i & 1ull) {
            ++m2l_ops;
            if (want_e4) entries.push_back(cand[P * FMM_CAND_MAX + i]);
          }
        if (want_e4) offs.push_back((int64_t)entries.size());
      }
    }
  }
  switch (what) {
    case FMM_X_NEAR_OWNERS:
    case FMM_X_E4_OWNERS: return copy_host(owners.data(), owners.size() * 4, host_buf, bytes, needed);
    case FMM_X_NEAR_OFFSETS:
    case FMM_X_E4_OFFSETS: return copy_host(offs.data(), offs.size() * 8, host_buf, bytes, needed);
    case FMM_X_NEAR_ENTRIES:
    case FMM_X_E4_ENTRIES: return copy_host(entries.data(), entries.size() * 4, host_buf, bytes, needed);
    case FMM_X_COUNTERS: {
      int64_t c[4] = {m2l_ops, p2p_pairs, ne_src, ne_tgt};
      return copy_host(c, sizeof(c), host_buf, bytes, needed);
    }
    default: return FMM_EBADCFG;
  }
}

}  // extern "C"
