// build.cu -- tree build on the device: keying (CellIndex), stable LSD radix sort by
// (leaf key, input index), leaf CSR offsets, cell centres and interaction lists.
//   keying      : PAPER.md P:207-250 (septree), P:342-364 (triangle), P:79 (Morton)
//   sort / CSR  : "Indexing: cell indices satisfy some order relation in memory"
//   lists       : P:101-111 Neighbors / NeighborsE4 (set-difference reading D1, from level 1: D2)
#include <limits.h>

#include <algorithm>

#include "fmm_internal.cuh"
#include "geometry.cuh"

DGeo dgeo(const Geo& g) {
  DGeo d;
  d.tiling = g.tiling;
  d.L = g.L;
  d.B = g.B;
  d.K = g.K;
  d.root_x = g.root_x;
  d.root_y = g.root_y;
  d.root_size = g.root_size;
  d.sept_A = g.sept_A;
  d.sept_Bc = g.sept_Bc;
  d.sept_D3r = g.sept_D3r;
  return d;
}

namespace {

// One 32-byte record (two double2, 32-byte aligned) moved by a single 256-bit global access
// (sm_100: LDG / STG .ENL2.256), so that a scattered record costs one L2 transaction per lane, not two.
__device__ __forceinline__ void st_rec(double2* __restrict__ rec, int64_t pos, double2 a, double2 b) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(rec + 2 * pos), "l"(__double_as_longlong(a.x)),
               "l"(__double_as_longlong(a.y)), "l"(__double_as_longlong(b.x)), "l"(__double_as_longlong(b.y))
               : "memory");
}
__device__ __forceinline__ void ld_rec(const double2* __restrict__ rec, int64_t pos, double2* a, double2* b) {
  long long x, y, z, w;
  asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(x), "=l"(y), "=l"(z), "=l"(w) : "l"(rec + 2 * pos));
  *a = make_double2(__longlong_as_double(x), __longlong_as_double(y));
  *b = make_double2(__longlong_as_double(z), __longlong_as_double(w));
}

// ------------------------------------------------------------------ keying
// key per point; out-of-domain points get the sentinel key K (sorted past every leaf)
// and report the minimal offending index.  (The leaf CSR comes from the sorted keys.)
// With hist != nullptr it also counts every leaf (the multi-rank global histogram), and with
// bin_cap > 0 (the bucket sort) it packs (x, y, u, input index) into one 32-byte record per point
// and drops it straight into the point's leaf bin, bins[k bin_cap + slot], the slot claimed by
// the same atomic that counts the leaf (one per distinct key of a warp; its lanes take consecutive
// slots in lane order); a point whose slot is past the bin's capacity is counted but not stored
// (the build then takes the LSD sort: k_sort_mode).
__global__ void __launch_bounds__(256) k_keys(DGeo g, const double2* __restrict__ xy, int64_t n,
                                              int64_t index_base, uint32_t* __restrict__ key, DevStatus* st,
                                              const double* __restrict__ u = nullptr,
                                              double2* __restrict__ bins = nullptr,
                                              int32_t* __restrict__ hist = nullptr, int bin_cap = 0) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = i < n;
  uint32_t k = 0xffffffffu;  // lanes past n: a key no point has (they form their own match group)
  double2 p = make_double2(0.0, 0.0);
  if (valid) {
    p = xy[i];
    if (!geo_key(g, p.x, p.y, &k)) {
      k = (uint32_t)g.K;
      atomicMin(&st->domain_bad, (unsigned long long)(index_base + i));
    }
    key[i] = k;
  }
  if (hist) {  // leaf histogram of every point, one atomic per distinct key of the warp
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
    if (!bin_cap) {
      if (valid && lane == leader) atomicAdd(&hist[k], __popc(peers));
      return;
    }
    int base = 0;
    if (valid && lane == leader) base = atomicAdd(&hist[k], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int slot = base + __popc(peers & ((1u << lane) - 1u));
    if (valid && slot < bin_cap) {
      st_rec(bins, (int64_t)k * bin_cap + slot, p, make_double2(u ? u[i] : 0.0, __longlong_as_double(i)));
    }
  }
}

// leaf CSR from the sorted keys: off[k] = #points with key < k, k = 0..K+1; position i
// (0..n) writes off[k] = i for prev < k <= cur, prev = sorted[i-1] (-1 at i = 0) and
// cur = sorted[i] (K+1 at i = n), so every entry is written exactly once
__global__ void __launch_bounds__(256) k_offsets(const uint32_t* __restrict__ sorted, int64_t n, int64_t K,
                                                 int32_t* __restrict__ off, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  // grid-stride (gated_grid): a gated-off launch costs one wave of blocks, not n / 256
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = i > 0 ? (int64_t)sorted[i - 1] : -1;
    const int64_t cur = i < n ? (int64_t)sorted[i] : K + 1;
    for (int64_t k = prev + 1; k <= cur; ++k) off[k] = (int32_t)i;
  }
}

// ------------------------------------------------------------------ scan (exclusive, int32)
constexpr int SCAN_T = 1024, SCAN_I = 8, SCAN_TILE = SCAN_T * SCAN_I;

__device__ inline int block_excl_scan(int v, int* total) {
  __shared__ int warp_tot[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive
  }
  __syncthreads();
  int before = w ? warp_tot[w - 1] : 0;
  *total = warp_tot[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before + x - v;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(const int32_t* __restrict__ in, int64_t n,
                                                         int32_t* __restrict__ bsum, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_I;
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k)
    if (base + k < n) s += in[base + k];
  int tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_block_sums(int32_t* bsum, int64_t nb, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  // single block, exclusive scan of up to SCAN_TILE block sums, in place
  int64_t base = threadIdx.x * SCAN_I;
  int v[SCAN_I], s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    v[k] = base + k < nb ? bsum[base + k] : 0;
    s += v[k];
  }
  int tot;
  int run = block_excl_scan(s, &tot);
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    if (base + k < nb) bsum[base + k] = run;
    run += v[k];
  }
}

__global__ void __launch_bounds__(SCAN_T) k_scan_apply(const int32_t* in, int64_t n, const int32_t* __restrict__ bsum,
                                                        int32_t* out, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_I;
  int v[SCAN_I], s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int tot;
  int run = block_excl_scan(s, &tot) + bsum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_I; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// ------------------------------------------------------------------ LSD radix sort (<= 10-bit digits)
// A tile of RS_TILE keys is split into RS_W warp segments of RS_SEG consecutive keys.  Ranks are
// stable: order = (warp segment, round, lane), from warp match masks and warp-private per-digit
// counters, so each tile needs only two block barriers per pass.
constexpr int RS_W = 8, RS_T = 32 * RS_W, RS_SEG = 512, RS_TILE = RS_W * RS_SEG, RS_MAXB = 10;

// lanes of the warp holding the same db-bit digit as this lane (valid lanes only): one ballot
// per digit bit (cheaper than match.any, whose latency bounded the sort)
__device__ __forceinline__ unsigned radix_peers(unsigned d, int db, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
  for (int b = 0; b < db; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

template <int SEG = RS_SEG>
__global__ void __launch_bounds__(RS_T) k_radix_upsweep(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                          int db, int32_t* __restrict__ tile_hist, int ntiles) {
  __shared__ int cnt[RS_W][1 << RS_MAXB];
  const int nb = 1 << db, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < nb; d += 32) cnt[w][d] = 0;
  __syncwarp();
  const int64_t seg0 = (int64_t)blockIdx.x * (RS_W * SEG) + (int64_t)w * SEG;
  const unsigned mask = (unsigned)nb - 1u;
  for (int r = 0; r < SEG / 32; ++r) {
    const int64_t i = seg0 + 32 * r + lane;
    const bool valid = i < n;
    const unsigned d = valid ? ((keys[i] >> shift) & mask) : 0u;
    const unsigned peers = radix_peers(d, db, valid);
    if (valid && lane == __ffs(peers) - 1) cnt[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nb; d += RS_T) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < RS_W; ++q) c += cnt[q][d];
    tile_hist[(int64_t)d * ntiles + blockIdx.x] = c;
  }
}

__global__ void __launch_bounds__(RS_T) k_radix_downsweep(const uint32_t* __restrict__ keys,
                                                            const int32_t* __restrict__ vals, int64_t n, int shift,
                                                            int db, const int32_t* __restrict__ tile_off, int ntiles,
                                                            uint32_t* __restrict__ keys_out,
                                                            int32_t* __restrict__ vals_out) {
  __shared__ int wb[RS_W][1 << RS_MAXB];  // per warp and digit: count, then running output position
  const int nb = 1 << db, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned mask = (unsigned)nb - 1u, lt = (1u << lane) - 1u;
  for (int d = lane; d < nb; d += 32) wb[w][d] = 0;
  __syncwarp();
  const int64_t seg0 = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * RS_SEG;
  // 1. per-warp digit counts of the warp's segment
  for (int r = 0; r < RS_SEG / 32; ++r) {
    const int64_t i = seg0 + 32 * r + lane;
    const bool valid = i < n;
    const unsigned d = valid ? ((keys[i] >> shift) & mask) : 0u;
    const unsigned peers = radix_peers(d, db, valid);
    if (valid && lane == __ffs(peers) - 1) wb[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 2. output base of each (warp, digit): the tile's offset of the digit + earlier warps
  for (int d = threadIdx.x; d < nb; d += RS_T) {
    int run = tile_off[(int64_t)d * ntiles + blockIdx.x];
#pragma unroll
    for (int q = 0; q < RS_W; ++q) {
      const int c = wb[q][d];
      wb[q][d] = run;
      run += c;
    }
  }
  __syncthreads();
  // 3. stable scatter in (round, lane) order within the warp's segment
  for (int r = 0; r < RS_SEG / 32; ++r) {
    const int64_t i = seg0 + 32 * r + lane;
    const bool valid = i < n;
    const uint32_t k = valid ? keys[i] : 0u;
    const unsigned d = valid ? ((k >> shift) & mask) : 0u;
    const unsigned peers = radix_peers(d, db, valid);
    int pos = 0;
    if (valid) pos = wb[w][d] + __popc(peers & lt);
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wb[w][d] += __popc(peers);
    if (valid) {
      keys_out[pos] = k;
      vals_out[pos] = vals ? vals[i] : (int32_t)i;
    }
    __syncwarp();
  }
}

// tile digit counts of the record sort: all of a thread's keys loaded first (one memory latency
// per tile), counted with shared-memory atomics (the counts do not depend on order)
__global__ void __launch_bounds__(RS_T) k_radix_count(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                        int db, int32_t* __restrict__ tile_hist, int ntiles,
                                                        int tile_elems, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  __shared__ int cnt[1 << RS_MAXB];
  const int nb = 1 << db;
  const unsigned mask = (unsigned)nb - 1u;
  for (int d = threadIdx.x; d < nb; d += RS_T) cnt[d] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * tile_elems;
  const int64_t t1 = min(n, t0 + tile_elems);
  for (int64_t i = t0 + threadIdx.x; i < t1; i += RS_T) atomicAdd(&cnt[(keys[i] >> shift) & mask], 1);
  __syncthreads();
  for (int d = threadIdx.x; d < nb; d += RS_T) tile_hist[(int64_t)d * ntiles + blockIdx.x] = cnt[d];
}

// The same stable scatter carrying the 32-byte record (x, y, u, input index) of each key
// instead of an index, so that the sorted sources come out of the last pass in place (no random
// gather after the sort), staged through shared memory: a tile of RR_TILE elements is first
// placed in digit order in shared memory (tile-local offsets of the digits + the stable rank),
// then written out by consecutive threads, so that the elements of one digit -- consecutive
// output positions -- leave in coalesced runs instead of one 16-byte store per element.
// FINAL: the last pass writes the record's fields to their SoA homes (sorted positions with a
// canonical +0 for a -0 coordinate, D13; strengths when su != NULL; the permutation) and the
// sorted keys (for the leaf CSR).  FIRST: the first pass forms the records from the caller's
// arrays (xy_in, u_in or NULL, the position as the input index) instead of reading them.
constexpr int RR_SEG = 256, RR_TILE = RS_W * RR_SEG;
constexpr size_t RR_SMEM = sizeof(int) * (RS_W + 2) * (1 << RS_MAXB) + sizeof(uint32_t) * RR_TILE +
                           2 * sizeof(double2) * RR_TILE;
template <bool FINAL, bool FIRST>
__global__ void __launch_bounds__(RS_T) k_radix_scatter_rec(const uint32_t* __restrict__ keys,
                                                              const double2* __restrict__ rec,
                                                              const double2* __restrict__ xy_in,
                                                              const double* __restrict__ u_in, int64_t n, int shift,
                                                              int db, const int32_t* __restrict__ tile_off,
                                                              int ntiles, uint32_t* __restrict__ keys_out,
                                                              double2* __restrict__ rec_out,
                                                              double2* __restrict__ sxy, double* __restrict__ su,
                                                              int32_t* __restrict__ perm, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  extern __shared__ double2 rr_smem[];
  double2* srec = rr_smem;                                   // [RR_TILE][2]
  uint32_t* skey = (uint32_t*)(srec + 2 * RR_TILE);          // [RR_TILE]
  int* wb = (int*)(skey + RR_TILE);                          // [RS_W][1 << RS_MAXB]
  int* loff = wb + RS_W * (1 << RS_MAXB);                    // tile-local digit starts
  int* goff = loff + (1 << RS_MAXB);                         // global - local offset per digit
  __shared__ int s_wsum[RS_W];
  const int nb = 1 << db, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned mask = (unsigned)nb - 1u, lt = (1u << lane) - 1u;
  for (int d = lane; d < nb; d += 32) wb[w * (1 << RS_MAXB) + d] = 0;
  __syncwarp();
  const int64_t tile0 = (int64_t)blockIdx.x * RR_TILE;
  const int64_t seg0 = tile0 + (int64_t)w * RR_SEG;
  // 0. every key and record of the warp's segment into registers at once (one memory latency
  // per tile instead of one per round)
  constexpr int NR = RR_SEG / 32;
  uint32_t kr[NR];
  double2 ra[NR], rb[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int64_t i = seg0 + 32 * r + lane;
    kr[r] = i < n ? keys[i] : 0u;
    if (FIRST) {
      ra[r] = i < n ? xy_in[i] : make_double2(0.0, 0.0);
      rb[r] = make_double2((i < n && u_in) ? u_in[i] : 0.0, __longlong_as_double(i));
    } else {
      ra[r] = rb[r] = make_double2(0.0, 0.0);
      if (i < n) ld_rec(rec, i, &ra[r], &rb[r]);
    }
  }
  // 1. per-warp digit counts
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const bool valid = seg0 + 32 * r + lane < n;
    const unsigned d = valid ? ((kr[r] >> shift) & mask) : 0u;
    const unsigned peers = radix_peers(d, db, valid);
    if (valid && lane == __ffs(peers) - 1) wb[w * (1 << RS_MAXB) + d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 2. per digit: each warp's rank base within the digit, and the tile count (into loff)
  for (int d = threadIdx.x; d < nb; d += RS_T) {
    int run = 0;
#pragma unroll
    for (int q = 0; q < RS_W; ++q) {
      const int c = wb[q * (1 << RS_MAXB) + d];
      wb[q * (1 << RS_MAXB) + d] = run;
      run += c;
    }
    loff[d] = run;
  }
  __syncthreads();
  // exclusive scan of the tile counts over the digits (RS_T threads x nb / RS_T digits)
  {
    const int per = (nb + RS_T - 1) / RS_T, d0 = threadIdx.x * per;
    int v[4], sum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = (k < per && d0 + k < nb) ? loff[d0 + k] : 0;
      sum += v[k];
    }
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[w] = x;
    __syncthreads();
    int base = 0;
    for (int q = 0; q < w; ++q) base += s_wsum[q];
    int run = base + x - sum;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < per && d0 + k < nb) {
        loff[d0 + k] = run;
        goff[d0 + k] = tile_off[(int64_t)(d0 + k) * ntiles + blockIdx.x] - run;
        run += v[k];
      }
  }
  __syncthreads();
  // 3. stage every element at its tile-local sorted position
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const bool valid = seg0 + 32 * r + lane < n;
    const unsigned d = valid ? ((kr[r] >> shift) & mask) : 0u;
    const unsigned peers = radix_peers(d, db, valid);
    int loc = 0;
    if (valid) loc = loff[d] + wb[w * (1 << RS_MAXB) + d] + __popc(peers & lt);
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wb[w * (1 << RS_MAXB) + d] += __popc(peers);
    if (valid) {
      skey[loc] = kr[r];
      srec[2 * loc] = ra[r];
      srec[2 * loc + 1] = rb[r];
    }
    __syncwarp();
  }
  __syncthreads();
  // 4. write out in tile-sorted order: runs of one digit go to consecutive positions
  const int cnt = (int)min((int64_t)RR_TILE, n - tile0);
  for (int j = threadIdx.x; j < cnt; j += RS_T) {
    const uint32_t k = skey[j];
    const int64_t g = goff[(k >> shift) & mask] + j;
    const double2 a = srec[2 * j], b = srec[2 * j + 1];
    keys_out[g] = k;
    if (FINAL) {
      sxy[g] = make_double2(__dadd_rn(a.x, 0.0), __dadd_rn(a.y, 0.0));  // -0 -> +0 (D13, p2p.cu)
      if (su) su[g] = b.x;
      perm[g] = (int32_t)__double_as_longlong(b.y);
    } else {
      st_rec(rec_out, g, a, b);
    }
  }
}

// ------------------------------------------------------------------ bucket sort (one rank)
// Stable order by (key, input index) in two streaming passes instead of two LSD radix passes:
// the keying kernel counts every leaf and drops each point's 32-byte record (x, y, u, input
// index) into its leaf's bin (LO_WARP_MAX records per leaf, slot = the count returned by the
// atomic: k_keys with bin_cap); the exclusive scan of the counts is the leaf CSR itself; and
// k_leaf_order restores input order inside each leaf (a warp ranks each record by counting the
// smaller input indices of its leaf) while writing the sorted SoA arrays and the permutation.
// The bins take the L2's atomic throughput per leaf counter and (K + 1) LO_WARP_MAX records of
// scratch, and the ranking is quadratic in the leaf size, so the bucket sort serves small leaves
// only: trees with more than LO_MEAN_MAX points per leaf on average, or with a leaf above
// LO_WARP_MAX points, take the LSD record sort (measured: DESIGN.md §8c).
constexpr int LO_WARP_MAX = 256;  // points of a leaf ordered by one warp = capacity of a leaf's bin
constexpr int LO_MEAN_MAX = 80;   // mean points per leaf above which the LSD sort is taken directly
constexpr size_t LO_BIN_BYTES_MAX = (size_t)4 << 30;  // bins of one point set (else the LSD sort)

__device__ __forceinline__ int rec_index(const double2* __restrict__ rec, int64_t pos) {
  return (int)__double_as_longlong(rec[2 * pos + 1].y);
}

// the record at bin position pos goes to sorted position o: coordinates with a canonical +0
// for a -0 (D13, p2p.cu), strength, input index
__device__ __forceinline__ void lo_write(const double2* __restrict__ rec, int64_t pos, int64_t o,
                                        double2* __restrict__ sxy, double* __restrict__ su,
                                        int32_t* __restrict__ perm) {
  double2 a, b;
  ld_rec(rec, pos, &a, &b);
  sxy[o] = make_double2(__dadd_rn(a.x, 0.0), __dadd_rn(a.y, 0.0));
  if (su) su[o] = b.x;
  perm[o] = (int)__double_as_longlong(b.y);
}

// one warp per bucket (K + 1 buckets: the leaves and the out-of-domain sentinel K): rank of each
// record = number of records of the bucket with a smaller input index (indices are distinct);
// the bucket's records sit in its bin from bb, its sorted range starts at b
template <int R>
__device__ __forceinline__ void lo_rank_warp(const int* __restrict__ sidx, int n, int lane, int64_t bb, int64_t b,
                                             const double2* __restrict__ rec, double2* __restrict__ sxy,
                                             double* __restrict__ su, int32_t* __restrict__ perm) {
  int mine[R], rank[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    mine[r] = lane + 32 * r < n ? sidx[lane + 32 * r] : INT_MAX;
    rank[r] = 0;
  }
  for (int j = 0; j < n; ++j) {
    const int v = sidx[j];
#pragma unroll
    for (int r = 0; r < R; ++r) rank[r] += v < mine[r];
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (lane + 32 * r < n) lo_write(rec, bb + lane + 32 * r, b + rank[r], sxy, su, perm);
}

__global__ void __launch_bounds__(256) k_leaf_order(int64_t nbuckets, const int32_t* __restrict__ off,
                                                    const double2* __restrict__ bins, double2* __restrict__ sxy,
                                                    double* __restrict__ su, int32_t* __restrict__ perm, const int32_t* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && *gate != gate_want) return;  // the other sort path runs (single_rank_keys_sort)
  __shared__ int sidx[8][LO_WARP_MAX];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k = blockIdx.x * 8ll + w;
  if (k >= nbuckets) return;
  const int64_t b = off[k];
  const int n = off[k + 1] - (int)b;
  if (n <= 0) return;  // (n <= LO_WARP_MAX: the gate)
  const int64_t bb = k * LO_WARP_MAX;  // the leaf's bin
  int* si = sidx[w];
  for (int e = lane; e < n; e += 32) si[e] = rec_index(bins, bb + e);
  __syncwarp();
  if (n <= 32)
    lo_rank_warp<1>(si, n, lane, bb, b, bins, sxy, su, perm);
  else if (n <= 64)
    lo_rank_warp<2>(si, n, lane, bb, b, bins, sxy, su, perm);
  else if (n <= 128)
    lo_rank_warp<4>(si, n, lane, bb, b, bins, sxy, su, perm);
  else
    lo_rank_warp<8>(si, n, lane, bb, b, bins, sxy, su, perm);
}

// largest bucket (leaves and the sentinel) of a count array
__global__ void __launch_bounds__(256) k_max_i32(const int32_t* __restrict__ v, int64_t n, int32_t* __restrict__ mx) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, v[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

// ------------------------------------------------------------------ gathers
// multi-rank: the kept sources gathered straight from the caller's arrays (no packed record:
// the rank keeps ~1/R of the points, so writing a record for every point would cost more)
__global__ void k_gather_src_in(const int32_t* __restrict__ perm, int64_t n, const double2* __restrict__ xy,
                                const double* __restrict__ u, double2* __restrict__ sxy, double* __restrict__ su) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = perm[i];
  const double2 v = xy[j];
  sxy[i] = make_double2(__dadd_rn(v.x, 0.0), __dadd_rn(v.y, 0.0));  // -0 -> +0 (D13, p2p.cu)
  su[i] = u[j];
}
__global__ void k_gather_xy(const int32_t* __restrict__ perm, int64_t n, const double2* __restrict__ xy,
                            double2* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = xy[perm[i]];
  out[i] = make_double2(__dadd_rn(v.x, 0.0), __dadd_rn(v.y, 0.0));  // -0 -> +0 (D13, p2p.cu)
}

// ------------------------------------------------------------------ centres (D12)
// level offsets of the all-level cell arrays (level l = cells [off[l], off[l+1]))
struct LevelOffsets {
  int64_t off[18];
  int nl;  // levels 0..nl-1
};
__device__ inline int level_of(const LevelOffsets& lo, int64_t gi) {
  int l = 0;
  while (l + 1 < lo.nl && gi >= lo.off[l + 1]) ++l;
  return l;
}

// every cell of every level in one launch (the small upper levels would each be a
// latency-bound launch of their own)
__global__ void k_centres(DGeo g, LevelOffsets lo, double2* __restrict__ out) {
  const int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gi >= lo.off[lo.nl]) return;
  const int l = level_of(lo, gi);
  out[gi] = geo_centre(g, l, gi - lo.off[l]);
}

// ------------------------------------------------------------------ interaction lists
__device__ inline int32_t cell_count(const int32_t* __restrict__ off, int64_t cell, int64_t span) {
  return off[(cell + 1) * span] - off[cell * span];
}

__device__ inline void sort_small(int64_t* v, int n) {
  for (int i = 1; i < n; ++i) {
    int64_t x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
}

// Candidates, one thread per parent P at level l-1: Children(P U Neighbors(P, l-1)) with
// sources, ascending (none when no child of P has targets of this rank).
// candidates of every parent cell P of levels 0..L-1 (children level l = level(P) + 1), one launch;
// cand / ncand are the all-level arrays indexed by the parent's global cell index
__global__ void k_cand_level(DGeo g, LevelOffsets lvo, const int32_t* __restrict__ soff,
                             const int32_t* __restrict__ toff, int32_t* __restrict__ cand_all,
                             int32_t* __restrict__ ncand_all, int64_t leaf_lo, int64_t leaf_hi) {
  const int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gi >= lvo.off[g.L]) return;  // parents live on levels 0..L-1
  const int l = level_of(lvo, gi) + 1;
  const int64_t P = gi - lvo.off[l - 1];
  int32_t* const cand = cand_all + lvo.off[l - 1] * FMM_CAND_MAX;
  int32_t* const ncand = ncand_all + lvo.off[l - 1];
  const int B = g.B;
  int64_t span_l = ipow_d(B, g.L - l), span_p = span_l * B;
  // parent's target range intersected with this rank's leaf range
  int64_t lo = P * span_p, hi = lo + span_p;
  bool has_t = (hi > leaf_lo && lo < leaf_hi) &&
               (toff[min(hi, leaf_hi)] - toff[max(lo, leaf_lo)] > 0);
  if (!has_t) {
    ncand[P] = 0;
    return;
  }
  int32_t* my = cand + P * FMM_CAND_MAX;
  // {P} U Neighbors(P) sorted (<= 13 cells); their children occupy disjoint ascending key
  // ranges [Q B, Q B + B), so emitting children in that order gives the ascending candidates
  int64_t pn[17];
  int npn = geo_neighbors(g, l - 1, P, pn);
  pn[npn++] = P;
  sort_small(pn, npn);
  int nc = 0;
  for (int q = 0; q < npn; ++q) {
    for (int ch = 0; ch < B; ++ch) {
      int64_t cc = pn[q] * B + ch;
      if (cell_count(soff, cc, span_l) > 0) my[nc++] = (int32_t)cc;
    }
  }
  ncand[P] = nc;
}

// E4 masks, one thread per cell t at level l: bit i set iff cand[parent][i] is not in
// {t} U Neighbors(t, l)  (NeighborsE4, reading D1); 0 when t has no targets.
// E4 masks of every cell of levels 1..L in one launch (after k_cand_level)
__global__ void k_e4mask_level(DGeo g, LevelOffsets lvo, const int32_t* __restrict__ toff,
                               const int32_t* __restrict__ cand_all, const int32_t* __restrict__ ncand_all,
                               unsigned long long* __restrict__ e4mask_all, int64_t leaf_lo, int64_t leaf_hi) {
  const int64_t gi = lvo.off[1] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gi >= lvo.off[g.L + 1]) return;
  const int l = level_of(lvo, gi);
  const int64_t t = gi - lvo.off[l];
  const int32_t* const cand = cand_all + lvo.off[l - 1] * FMM_CAND_MAX;
  const int32_t* const ncand = ncand_all + lvo.off[l - 1];
  unsigned long long* const e4mask = e4mask_all + lvo.off[l];
  int64_t span_l = ipow_d(g.B, g.L - l);
  int64_t tl = t * span_l, th = tl + span_l;
  bool t_has = (th > leaf_lo && tl < leaf_hi) && (toff[min(th, leaf_hi)] - toff[max(tl, leaf_lo)] > 0);
  unsigned long long mask = 0ull;
  if (t_has) {
    const int64_t P = t / g.B;
    const int nc = ncand[P];
    const int32_t* c = cand + P * FMM_CAND_MAX;
    int64_t nb[17];
    int nn = geo_neighbors(g, l, t, nb);
    nb[nn++] = t;
    sort_small(nb, nn);
    // both lists ascending: one merge pass marks the candidates outside {t} U Neighbors(t)
    int k = 0;
    for (int i = 0; i < nc; ++i) {
      const int64_t ci = c[i];
      while (k < nn && nb[k] < ci) ++k;
      if (!(k < nn && nb[k] == ci)) mask |= 1ull << i;
    }
  }
  e4mask[t] = mask;
}

// near(t) = ({t} U Neighbors(t, L)) with sources, ascending
__device__ void near_of(const DGeo& g, int64_t t, const int32_t* __restrict__ soff, int32_t* __restrict__ near,
                        int32_t* __restrict__ nnear) {
  int64_t nb[17];
  int nn = geo_neighbors(g, g.L, t, nb);
  nb[nn++] = t;
  int64_t v[17];
  int k = 0;
  for (int i = 0; i < nn; ++i)
    if (soff[nb[i] + 1] - soff[nb[i]] > 0) v[k++] = nb[i];
  sort_small(v, k);
  for (int i = 0; i < k; ++i) near[t * FMM_NEAR_MAX + i] = (int32_t)v[i];
  nnear[t] = k;
}

__global__ void k_near(DGeo g, const int32_t* __restrict__ soff, const int32_t* __restrict__ toff,
                       int32_t* __restrict__ near, int32_t* __restrict__ nnear, int64_t leaf_lo, int64_t leaf_hi) {
  int64_t t = leaf_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= leaf_hi) return;
  if (toff[t + 1] - toff[t] == 0) {
    nnear[t] = 0;
    return;
  }
  near_of(g, t, soff, near, nnear);
}

// ------------------------------------------------------------------ multi-rank selection
// source leaves this rank keeps: its own leaf range [lo, hi) (it computes their P2M) and every
// near source leaf of its own target leaves (the P2P halo); byte flags (idempotent
// stores), packed to a bitmask below
__global__ void k_halo_flags(int64_t lo, int64_t hi, const int32_t* __restrict__ gtoff,
                             const int32_t* __restrict__ near, const int32_t* __restrict__ nnear,
                             uint8_t* __restrict__ flag) {
  const int64_t t = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= hi) return;
  flag[t] = 1;
  if (gtoff[t + 1] == gtoff[t]) return;
  for (int q = 0; q < nnear[t]; ++q) flag[near[t * FMM_NEAR_MAX + q]] = 1;
}

// the keep flags (bytes) packed into the leaf bitmask, one word per warp
__global__ void __launch_bounds__(256) k_pack_bits(int64_t K, const uint8_t* __restrict__ flag,
                                                   uint32_t* __restrict__ bits) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const unsigned word = __ballot_sync(0xffffffffu, t <= K && flag[t]);
  if ((threadIdx.x & 31) == 0 && t <= K) bits[t >> 5] = word;
}

// Stable single-pass compaction of the kept points (input order, so that the sort by key then
// gives the (key, input index) order of the single-rank tree).  Keep predicate: the point's
// leaf bit is set (bits != NULL: sources), else its leaf lies in [lo, hi) (distinct targets).
// Tiles of CP_TILE keys are taken in ticket order; each publishes its kept count and finds its
// output offset by a decoupled look-back over the earlier tiles' status words (state in bits
// 62-63: 1 = tile count, 2 = inclusive prefix).  The leaf bitmask (32 KB for 2^18 leaves) sits in
// shared memory when it fits, so the per-point lookups do not go to L2.
constexpr int CP_T = 256, CP_V = 16, CP_TILE = CP_T * CP_V;
constexpr unsigned long long CP_AGG = 1ull << 62, CP_INC = 2ull << 62, CP_CNT = (1ull << 62) - 1;
__global__ void __launch_bounds__(CP_T) k_select_compact(const uint32_t* __restrict__ key, int64_t n,
                                                         const uint32_t* __restrict__ bits, int nwords_smem,
                                                         int64_t lo, int64_t hi, unsigned long long* tstat,
                                                         int32_t* ticket, uint32_t* __restrict__ ckey,
                                                         int32_t* __restrict__ cidx, int64_t* __restrict__ nout) {
  extern __shared__ uint32_t s_bits[];
  __shared__ int s_tile;
  __shared__ int s_warp[CP_T / 32];
  __shared__ long long s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // persistent blocks: the bitmask is staged once per block, tiles are taken by ticket
  for (int i = tid; i < nwords_smem; i += CP_T) s_bits[i] = bits[i];
  const uint32_t* bt = nwords_smem > 0 ? s_bits : bits;
  const int64_t ntiles = (n + CP_TILE - 1) / CP_TILE;
  while (true) {
    __syncthreads();  // s_bits staged / the previous tile's shared words consumed
    if (tid == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int tile = s_tile;
    if (tile >= ntiles) break;
    const int64_t base = (int64_t)tile * CP_TILE + (int64_t)tid * CP_V;
    uint32_t k[CP_V];
    unsigned keep = 0;
    if (base + CP_V <= n) {
      const uint4* kp = (const uint4*)(key + base);
#pragma unroll
      for (int v = 0; v < CP_V / 4; ++v) {
        const uint4 q = kp[v];
        k[4 * v] = q.x, k[4 * v + 1] = q.y, k[4 * v + 2] = q.z, k[4 * v + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int v = 0; v < CP_V; ++v) k[v] = base + v < n ? key[base + v] : 0xffffffffu;
    }
#pragma unroll
    for (int v = 0; v < CP_V; ++v) {
      bool kp;
      if (k[v] == 0xffffffffu) kp = false;
      else if (bits) kp = (bt[k[v] >> 5] >> (k[v] & 31)) & 1u;
      else kp = (int64_t)k[v] >= lo && (int64_t)k[v] < hi;
      keep |= (unsigned)kp << v;
    }
    // block exclusive scan of the per-thread kept counts
    const int c = __popc(keep);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int i = 0; i < CP_T / 32; ++i) {
      if (i < w) wbase += s_warp[i];
      total += s_warp[i];
    }
    const int excl = wbase + x - c;
    // decoupled look-back by warp 0: 32 earlier tiles per round, summing counts down to the
    // nearest tile that has published its inclusive prefix
    if (w == 0) {
      if (lane == 0) atomicExch(&tstat[tile], (tile == 0 ? CP_INC : CP_AGG) | (unsigned long long)total);
      long long prefix = 0;
      for (int64_t j = tile - 1; j >= 0; j -= 32) {
        const int64_t idx = j - lane;
        unsigned long long v = CP_INC;  // before tile 0: an inclusive prefix of 0
        if (idx >= 0) {
          do {
            v = *(volatile unsigned long long*)&tstat[idx];
          } while ((v >> 62) == 0);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int first = inc ? __ffs(inc) - 1 : 32;
        long long c_ = lane <= first ? (long long)(v & CP_CNT) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c_ += __shfl_xor_sync(0xffffffffu, c_, o);
        prefix += c_;
        if (inc) break;
      }
      if (lane == 0) {
        if (tile > 0) atomicExch(&tstat[tile], CP_INC | (unsigned long long)(prefix + total));
        s_prefix = prefix;
        if (tile == ntiles - 1) *nout = prefix + total;
      }
    }
    __syncthreads();
    int64_t pos = s_prefix + excl;
#pragma unroll
    for (int v = 0; v < CP_V; ++v)
      if ((keep >> v) & 1u) {
        ckey[pos] = k[v];
        cidx[pos] = (int32_t)(base + v);
        ++pos;
      }
  }
}

// leaf CSR of a rank-local sorted key set (which skips whole key ranges): off[k] = lower bound
// of k in the sorted keys, k = 0..K+1 (binary search per leaf; k_offsets' one-thread gap fill
// would serialise over the skipped ranges)
__global__ void __launch_bounds__(256) k_offsets_search(const uint32_t* __restrict__ sorted, int64_t n, int64_t K,
                                                        int32_t* __restrict__ off) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k > K + 1) return;
  int64_t a = 0, b = n;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if ((int64_t)sorted[mid] < k) a = mid + 1;
    else b = mid;
  }
  off[k] = (int32_t)a;
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
// grid of a grid-stride kernel that may be gated off on the device: at most 8 blocks per SM
inline unsigned gated_grid(int64_t n, int t) { return (unsigned)std::min<int64_t>((n + t - 1) / t, 148 * 8); }

}  // namespace

// ====================================================================== host entry points
size_t fmm_scan_scratch_bytes(int64_t n) {
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  return (size_t)(nb + 32) * sizeof(int32_t);
}

// gate (device int, optional): the scan runs only when *gate == gate_want (build.cu's sort paths)
static int device_scan_gated(const int32_t* in, int32_t* out, int64_t n, void* scratch, size_t scratch_bytes,
                             cudaStream_t s, int64_t* launches, const int32_t* gate, int gate_want) {
  if (n <= 0) return FMM_OK;
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb > SCAN_TILE || scratch_bytes < fmm_scan_scratch_bytes(n)) return FMM_EBADCFG;
  int32_t* bsum = (int32_t*)scratch;
  k_scan_reduce<<<(unsigned)nb, SCAN_T, 0, s>>>(in, n, bsum, gate, gate_want);
  k_scan_block_sums<<<1, SCAN_T, 0, s>>>(bsum, nb, gate, gate_want);
  k_scan_apply<<<(unsigned)nb, SCAN_T, 0, s>>>(in, n, bsum, out, gate, gate_want);
  *launches += 3;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_device_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* scratch, size_t scratch_bytes,
                        cudaStream_t s, int64_t* launches) {
  return device_scan_gated(in, out, n, scratch, scratch_bytes, s, launches, nullptr, 0);
}

int64_t fmm_scan_max_entries() { return (int64_t)SCAN_TILE * SCAN_TILE; }

static int key_bits(int64_t K) {  // keys are 0..K (K = sentinel)
  int b = 1;
  while (((int64_t)1 << b) <= K) ++b;
  return b;
}

// sort (key, value) pairs stably, values = iota (vals0 == NULL) or vals0[i]; writes the
// permutation (sorted position -> value, i.e. input index) and the leaf CSR off[0..K+1] from
// the sorted keys
static int radix_sort_perm(fmm_tree_s* t, const uint32_t* keys, int64_t n, int32_t* perm, int32_t* off,
                           const int32_t* vals0 = nullptr) {
  if (n == 0) {
    FMM_CUDA_TRY(cudaMemsetAsync(off, 0, sizeof(int32_t) * (t->g.K + 2), t->stream));
    return FMM_OK;
  }
  cudaStream_t s = t->stream;
  const int bits = key_bits(t->g.K);
  const int passes = (bits + RS_MAXB - 1) / RS_MAXB;
  const int ntiles = (int)((n + RS_TILE - 1) / RS_TILE);
  const int64_t nhist = ((int64_t)1 << ((bits + passes - 1) / passes)) * ntiles;
  // scratch: kA kB (n u32), vA (n i32), hist (nhist), scan scratch
  size_t need = (size_t)n * 4 * 3 + (size_t)nhist * 4 + fmm_scan_scratch_bytes(nhist) + 256;
  if (t->scratch_bytes < need) {
    if (t->scratch) cudaFreeAsync(t->scratch, s);
    t->scratch = nullptr;
    FMM_CUDA_TRY(cudaMallocAsync(&t->scratch, need, s));
    t->scratch_bytes = need;
  }
  char* p = (char*)t->scratch;
  uint32_t* kA = (uint32_t*)p;
  p += (size_t)n * 4;
  uint32_t* kB = (uint32_t*)p;
  p += (size_t)n * 4;
  int32_t* vA = (int32_t*)p;
  p += (size_t)n * 4;
  int32_t* hist = (int32_t*)p;
  p += (size_t)nhist * 4;
  void* sscr = p;
  const uint32_t* kin = keys;
  const int32_t* vin = vals0;  // iota on the first pass when NULL
  int shift = 0;
  for (int ps = 0; ps < passes; ++ps) {
    // balanced digit widths: the first (bits % passes) passes take one more bit
    const int db = bits / passes + (ps < bits % passes ? 1 : 0);
    const int64_t nh = ((int64_t)1 << db) * ntiles;
    uint32_t* kout = (ps % 2 == 0) ? kA : kB;
    // values alternate between vA and perm such that the last pass writes perm
    int32_t* vout = ((passes - 1 - ps) % 2 == 0) ? perm : vA;
    k_radix_upsweep<<<ntiles, RS_T, 0, s>>>(kin, n, shift, db, hist, ntiles);
    int e = fmm_device_scan_i32(hist, hist, nh, sscr, fmm_scan_scratch_bytes(nh), s, &t->launches);
    if (e) return e;
    k_radix_downsweep<<<ntiles, RS_T, 0, s>>>(kin, vin, n, shift, db, hist, ntiles, kout, vout);
    t->launches += 2;
    FMM_CUDA_TRY(cudaGetLastError());
    kin = kout;
    vin = vout;
    shift += db;
  }
  if (t->cfg.nranks > 1)
    k_offsets_search<<<blocks_for(t->g.K + 2, 256), 256, 0, s>>>(kin, n, t->g.K, off);
  else
    k_offsets<<<gated_grid(n + 1, 256), 256, 0, s>>>(kin, n, t->g.K, off);
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

// multi-rank: global leaf counts of every rank's points, near lists of every
// leaf, the work-balanced leaf range of this rank (one host sync), its halo of near source
// leaves, and the stable compaction of the points it keeps (a second host sync reads their
// counts).  ckey / cidx (n + m entries each) receive the kept keys and input indices: sources
// first, then targets (distinct-target trees).
// stable LSD radix sort of (key, 32-byte record) pairs of one rank's points: the first pass forms
// the records (x, y, u, input index) from the caller's arrays, they move with the keys through
// every pass and the last pass writes the sorted SoA arrays and the permutation; then the leaf
// CSR off[0..K+1] from the sorted keys
// gate (device int, optional): every kernel of the sort runs only when *gate == 1 (the LSD path of
// single_rank_keys_sort, decided on the device)
static int radix_sort_records(fmm_tree_s* t, const uint32_t* keys, const double2* xy_in, const double* u_in,
                              int64_t n, double2* xy_out, double* u_out, int32_t* perm, int32_t* off,
                              const int32_t* gate = nullptr) {
  cudaStream_t s = t->stream;
  if (n == 0) {
    FMM_CUDA_TRY(cudaMemsetAsync(off, 0, sizeof(int32_t) * (t->g.K + 2), s));
    return FMM_OK;
  }
  const int bits = key_bits(t->g.K);
  const int passes = (bits + RS_MAXB - 1) / RS_MAXB;
  const int ntiles = (int)((n + RR_TILE - 1) / RR_TILE);
  const int64_t nhist = ((int64_t)1 << ((bits + passes - 1) / passes)) * ntiles;
  // per device (a process may drive several GPUs)
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter_rec<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RR_SMEM));
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter_rec<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RR_SMEM));
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter_rec<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RR_SMEM));
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_radix_scatter_rec<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RR_SMEM));
  // scratch: kA kB (n u32), record ping-pong (n x 32 B each: one buffer for two passes, two for
  // more), hist, scan scratch
  const int nrec = passes > 2 ? 2 : (passes > 1 ? 1 : 0);
  const size_t rec_bytes = (size_t)n * 32;
  const size_t need = 256 + (size_t)n * 8 + 256 + nrec * (rec_bytes + 256) + (size_t)nhist * 4 +
                      fmm_scan_scratch_bytes(nhist) + 256;
  if (t->scratch_bytes < need) {
    if (t->scratch) cudaFreeAsync(t->scratch, s);
    t->scratch = nullptr;
    FMM_CUDA_TRY(cudaMallocAsync(&t->scratch, need, s));
    t->scratch_bytes = need;
  }
  char* p = (char*)t->scratch;
  auto take = [&](size_t b) {
    char* q = p;
    p += (b + 255) & ~(size_t)255;
    return q;
  };
  uint32_t* kA = (uint32_t*)take((size_t)n * 4);
  uint32_t* kB = (uint32_t*)take((size_t)n * 4);
  double2* rA = nrec > 0 ? (double2*)take(rec_bytes) : nullptr;
  double2* rB = nrec > 1 ? (double2*)take(rec_bytes) : nullptr;
  int32_t* hist = (int32_t*)take((size_t)nhist * 4);
  void* sscr = p;
  const uint32_t* kin = keys;
  const double2* rin = nullptr;
  int shift = 0;
  for (int ps = 0; ps < passes; ++ps) {
    const int db = bits / passes + (ps < bits % passes ? 1 : 0);
    const int64_t nh = ((int64_t)1 << db) * ntiles;
    uint32_t* kout = (ps % 2 == 0) ? kA : kB;
    double2* rout = (ps % 2 == 0) ? rA : rB;
    k_radix_count<<<ntiles, RS_T, 0, s>>>(kin, n, shift, db, hist, ntiles, RR_TILE, gate, 1);
    int e = device_scan_gated(hist, hist, nh, sscr, fmm_scan_scratch_bytes(nh), s, &t->launches, gate, 1);
    if (e) return e;
    const bool fin = ps == passes - 1;
    auto kern = fin ? (ps == 0 ? k_radix_scatter_rec<true, true> : k_radix_scatter_rec<true, false>)
                    : (ps == 0 ? k_radix_scatter_rec<false, true> : k_radix_scatter_rec<false, false>);
    kern<<<ntiles, RS_T, RR_SMEM, s>>>(kin, rin, xy_in, u_in, n, shift, db, hist, ntiles, kout, fin ? nullptr : rout,
                                       fin ? xy_out : nullptr, fin ? u_out : nullptr, fin ? perm : nullptr, gate, 1);
    t->launches += 2;
    FMM_CUDA_TRY(cudaGetLastError());
    kin = kout;
    rin = rout;
    shift += db;
  }
  k_offsets<<<gated_grid(n + 1, 256), 256, 0, s>>>(kin, n, t->g.K, off, gate, 1);
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

static int multi_rank_select(fmm_tree_s* t, uint32_t* ckey, int32_t* cidx, int64_t* dcount) {
  cudaStream_t s = t->stream;
  const Geo& G = t->g;
  const int64_t K = G.K;
  // global histograms (made by the keying kernels) -> exclusive scans: gsoff[k] = #points with
  // key < k, k = 0..K+1
  const size_t sb = fmm_scan_scratch_bytes(K + 2);
  void* sscr = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync(&sscr, sb, s));
  int e = fmm_device_scan_i32(t->gsoff, t->gsoff, K + 2, sscr, sb, s, &t->launches);
  if (!e && !G.self_mode) e = fmm_device_scan_i32(t->gtoff, t->gtoff, K + 2, sscr, sb, s, &t->launches);
  cudaFreeAsync(sscr, s);
  if (e) return e;
  FMM_CUDA_TRY(cudaGetLastError());
  // near lists (global emptiness) and the partition
  e = fmm_stage_near_partition(t);
  if (e) return e;
  // halo flags of the source leaves (bytes, then a bitmask), then stable compactions of the kept
  // points
  const int64_t nwords = (K + 1 + 31) / 32;
  uint32_t* bits = (uint32_t*)t->lflag;
  uint8_t* flag8 = (uint8_t*)(bits + nwords);
  FMM_CUDA_TRY(cudaMemsetAsync(flag8, 0, K + 1, s));
  if (t->leaf_hi > t->leaf_lo)
    k_halo_flags<<<blocks_for(t->leaf_hi - t->leaf_lo, 128), 128, 0, s>>>(t->leaf_lo, t->leaf_hi, t->gtoff,
                                                                          t->near, t->nnear, flag8);
  k_pack_bits<<<blocks_for(K + 1, 256), 256, 0, s>>>(K, flag8, bits);
  t->launches += 2;
  // the bitmask goes to shared memory when it fits (<= 160 KB: 1.3M leaves)
  const int smem_words = nwords * 4 <= 160 * 1024 ? (int)nwords : 0;
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_select_compact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    std::max(smem_words * 4, 1)));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nt_s = (t->n + CP_TILE - 1) / CP_TILE;
  const int64_t nt_t = G.self_mode ? 0 : (t->m + CP_TILE - 1) / CP_TILE;
  unsigned long long* tstat = nullptr;  // tile status words of both compactions + 2 tickets
  const size_t stat_bytes = sizeof(unsigned long long) * (nt_s + nt_t + 2);
  FMM_CUDA_TRY(cudaMallocAsync((void**)&tstat, stat_bytes, s));
  FMM_CUDA_TRY(cudaMemsetAsync(tstat, 0, stat_bytes, s));
  FMM_CUDA_TRY(cudaMemsetAsync(dcount, 0, 2 * sizeof(int64_t), s));
  int32_t* tickets = (int32_t*)(tstat + nt_s + nt_t);
  const unsigned grid_s = (unsigned)std::min<int64_t>(nt_s, 2 * nsm), grid_t = (unsigned)std::min<int64_t>(nt_t, 4 * nsm);
  if (nt_s > 0) {
    k_select_compact<<<grid_s, CP_T, smem_words * 4, s>>>(t->skey, t->n, bits, smem_words, 0, 0, tstat,
                                                                  tickets, ckey, cidx, dcount);
    t->launches++;
  }
  if (nt_t > 0) {
    k_select_compact<<<grid_t, CP_T, 0, s>>>(t->tkey, t->m, nullptr, 0, t->leaf_lo, t->leaf_hi,
                                                     tstat + nt_s, tickets + 1, ckey + t->n, cidx + t->n,
                                                     dcount + 1);
    t->launches++;
  }
  cudaFreeAsync(tstat, s);
  FMM_CUDA_TRY(cudaGetLastError());
  int64_t h[2] = {0, 0};
  FMM_CUDA_TRY(cudaMemcpyAsync(h, dcount, sizeof(h), cudaMemcpyDeviceToHost, s));
  FMM_CUDA_TRY(cudaStreamSynchronize(s));
  t->n_loc = h[0];
  t->m_loc = G.self_mode ? h[0] : h[1];
  return FMM_OK;
}

// mode = 1 (LSD record sort) when some leaf holds more than LO_WARP_MAX points, else 0 (bucket)
__global__ void k_sort_mode(const int32_t* __restrict__ mx, int32_t* __restrict__ mode) {
  *mode = *mx > LO_WARP_MAX ? 1 : 0;
}

// one rank (DESIGN.md §7 "Build"), per point set: the LSD record sort when the leaves hold more
// than LO_MEAN_MAX points on average, the set is small or the leaf bins would not fit (host
// decisions); else keys with leaf counts and the records dropped into leaf bins, the leaf CSR from
// the counts' scan, and both sorts enqueued with every kernel gated by a device mode word -- the
// bucket sort's ordering pass when no leaf holds more than LO_WARP_MAX points, else the LSD record
// sort -- so that the build never waits on the device from the host.  FMM_SORT_LSD=1 forces the
// LSD sort.
static int single_rank_keys_sort(fmm_tree_s* t) {
  cudaStream_t s = t->stream;
  const Geo& G = t->g;
  DGeo g = dgeo(G);
  const int64_t K = G.K, nb = K + 2;
  const int nsets = G.self_mode ? 1 : 2;
  const int64_t cnt[2] = {t->n, G.self_mode ? 0 : t->m};
  t->n_loc = t->n;  // one rank keeps every point
  t->m_loc = t->m;
  const char* force = getenv("FMM_SORT_LSD");
  const bool force_lsd = force && force[0] == '1';
  const size_t bin_bytes = (size_t)(K + 1) * LO_WARP_MAX * 32;
  bool lsd[2];
  // small point sets (<= 2^20: launch-bound builds) skip the gated pair of paths
  for (int k = 0; k < 2; ++k)
    lsd[k] = force_lsd || cnt[k] > LO_MEAN_MAX * K || cnt[k] <= (1 << 20) || bin_bytes > LO_BIN_BYTES_MAX;
  // scratch per point set: counts (K + 2) | scan scratch; then two maxima and two mode words
  const size_t sscan = fmm_scan_scratch_bytes(nb);
  const size_t hb = ((size_t)nb * 4 + 255) / 256 * 256;
  const size_t per = hb + (sscan + 255) / 256 * 256;
  char* buf = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&buf, nsets * per + 256, s));
  int32_t* mx = (int32_t*)(buf + nsets * per);
  int32_t* mode = mx + 2;
  FMM_CUDA_TRY(cudaMemsetAsync(buf, 0, nsets * per + 256, s));
  auto hist = [&](int k) { return (int32_t*)(buf + k * per); };
  auto sscr = [&](int k) { return (void*)(buf + k * per + hb); };
  const double2* xy[2] = {(const double2*)t->src_xy_in, (const double2*)t->tgt_xy_in};
  const double* u[2] = {t->src_u_in, nullptr};
  uint32_t* keys[2] = {t->skey, t->tkey};
  int32_t* off[2] = {t->soff, t->toff};
  double2* xy_out[2] = {t->sxy, t->txy};
  double* u_out[2] = {t->su, nullptr};
  int32_t* perm[2] = {t->sperm, t->tperm};
  double2* bins[2] = {nullptr, nullptr};  // leaf bins (bucket sort)
  for (int k = 0; k < nsets; ++k)
    if (cnt[k] > 0) {
      if (!lsd[k]) FMM_CUDA_TRY(cudaMallocAsync((void**)&bins[k], bin_bytes, s));
      // LSD: keys only (its first pass forms the records); bucket: keys + counts + records into the bins
      k_keys<<<blocks_for(cnt[k], 256), 256, 0, s>>>(g, xy[k], cnt[k], k ? t->n : 0, keys[k], t->status, u[k],
                                                      lsd[k] ? nullptr : bins[k], lsd[k] ? nullptr : hist(k),
                                                      lsd[k] ? 0 : LO_WARP_MAX);
      t->launches++;
    }
  FMM_CUDA_TRY(cudaGetLastError());
  if (t->timing) cudaEventRecord(t->ev[8], s);
  if (t->timing) cudaEventRecord(t->ev[9], s);
  int e = FMM_OK;
  for (int k = 0; k < nsets && !e; ++k) {
    if (cnt[k] == 0) {
      FMM_CUDA_TRY(cudaMemsetAsync(off[k], 0, sizeof(int32_t) * nb, s));
      continue;
    }
    if (lsd[k]) {
      e = radix_sort_records(t, keys[k], xy[k], u[k], cnt[k], xy_out[k], u_out[k], perm[k], off[k]);
      continue;
    }
    e = fmm_device_scan_i32(hist(k), off[k], nb, sscr(k), sscan, s, &t->launches);
    if (e) break;
    k_max_i32<<<64, 256, 0, s>>>(hist(k), K + 1, mx + k);
    k_sort_mode<<<1, 1, 0, s>>>(mx + k, mode + k);
    t->launches += 2;
    // mode 1: the LSD record sort (its offsets overwrite the same CSR)
    e = radix_sort_records(t, keys[k], xy[k], u[k], cnt[k], xy_out[k], u_out[k], perm[k], off[k], mode + k);
    if (e) break;
    // mode 0: the bucket sort's ordering pass over the bins
    k_leaf_order<<<blocks_for(K + 1, 8), 256, 0, s>>>(K + 1, off[k], bins[k], xy_out[k], u_out[k], perm[k], mode + k, 0);
    t->launches++;
    FMM_CUDA_TRY(cudaGetLastError());
  }
  for (int k = 0; k < nsets; ++k)
    if (bins[k]) cudaFreeAsync(bins[k], s);
  cudaFreeAsync(buf, s);
  return e;
}

int fmm_stage_keys_sort(fmm_tree_s* t) {
  if (t->cfg.nranks <= 1) return single_rank_keys_sort(t);
  // multi-rank: keys of every point with the global leaf counts, the rank's
  // selection (compacted keys + input indices of the kept points), their stable radix sort,
  // then the kept points gathered from the caller's arrays
  cudaStream_t s = t->stream;
  const Geo& G = t->g;
  DGeo g = dgeo(G);
  FMM_CUDA_TRY(cudaMemsetAsync(t->gsoff, 0, sizeof(int32_t) * (G.K + 2), s));
  if (!G.self_mode) FMM_CUDA_TRY(cudaMemsetAsync(t->gtoff, 0, sizeof(int32_t) * (G.K + 2), s));
  if (t->n > 0) {
    k_keys<<<blocks_for(t->n, 256), 256, 0, s>>>(g, (const double2*)t->src_xy_in, t->n, 0, t->skey, t->status,
                                                  nullptr, nullptr, t->gsoff);
    t->launches++;
  }
  if (!G.self_mode && t->m > 0) {
    k_keys<<<blocks_for(t->m, 256), 256, 0, s>>>(g, (const double2*)t->tgt_xy_in, t->m, t->n, t->tkey, t->status,
                                                  nullptr, nullptr, t->gtoff);
    t->launches++;
  }
  FMM_CUDA_TRY(cudaGetLastError());
  if (t->timing) cudaEventRecord(t->ev[8], s);
  const int64_t tot = t->n + (G.self_mode ? 0 : t->m);
  char* buf = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&buf, (size_t)tot * 8 + 256, s));
  uint32_t* ckey = (uint32_t*)buf;
  int32_t* cidx = (int32_t*)(buf + (size_t)tot * 4);
  int64_t* dcount = (int64_t*)(buf + (size_t)tot * 8);
  int e = multi_rank_select(t, ckey, cidx, dcount);
  if (t->timing) cudaEventRecord(t->ev[9], s);
  // stable sorts of the compacted (key, input index) pairs; leaf CSR offsets from the sorted keys
  if (!e) e = radix_sort_perm(t, ckey, t->n_loc, t->sperm, t->soff, cidx);
  if (!e && !G.self_mode) e = radix_sort_perm(t, ckey + t->n, t->m_loc, t->tperm, t->toff, cidx + t->n);
  cudaFreeAsync(buf, s);
  if (e) return e;
  if (t->n_loc > 0) {
    k_gather_src_in<<<blocks_for(t->n_loc, 256), 256, 0, s>>>(t->sperm, t->n_loc, (const double2*)t->src_xy_in,
                                                               t->src_u_in, t->sxy, t->su);
    t->launches++;
  }
  if (!G.self_mode && t->m_loc > 0) {
    k_gather_xy<<<blocks_for(t->m_loc, 256), 256, 0, s>>>(t->tperm, t->m_loc, (const double2*)t->tgt_xy_in, t->txy);
    t->launches++;
  }
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

namespace {
// estimated evaluation work of each leaf (P2P pairs + per-target L2P + per-leaf downward),
// summed over blocks of FMM_PART_BLOCK leaves (the multi-rank partition)
// Work estimate of leaf t: w_t = n_t^tgt * sum_{s in near(t)} n_s^src (its near-field pairs)
// + 2 (p+1) n_t^tgt (L2P) + 40 (p+1)^2 (its M2L), from the global counts and the near lists of
// every leaf; summed per block of FMM_PART_BLOCK (= 32, one warp) leaves.  Clustered inputs
// need both: a few dense leaves carry a large share of the work, and their neighbours' counts
// differ from their own.
__global__ void k_block_work(int64_t K, const int32_t* __restrict__ soff, const int32_t* __restrict__ toff,
                             const int32_t* __restrict__ near, const int32_t* __restrict__ nnear, int p,
                             double* __restrict__ bw) {
  const int64_t leaf = blockIdx.x * (int64_t)FMM_PART_BLOCK + threadIdx.x;
  double w = 0.0;
  if (leaf < K) {
    const int nt = toff[leaf + 1] - toff[leaf];
    if (nt > 0) {
      int64_t ns = 0;
      for (int q = 0; q < nnear[leaf]; ++q) {
        const int sl = near[leaf * FMM_NEAR_MAX + q];
        ns += soff[sl + 1] - soff[sl];
      }
      w = (double)nt * (double)ns + 2.0 * (p + 1) * nt + 40.0 * (p + 1) * (p + 1);
    }
  }
  static_assert(FMM_PART_BLOCK == 32, "one warp per work block");
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if (threadIdx.x == 0) bw[blockIdx.x] = w;
}

}  // namespace

// near lists of every leaf (global emptiness); nranks > 1: then the work-balanced leaf range of
// this rank (one host sync)
int fmm_stage_near_partition(fmm_tree_s* t) {
  cudaStream_t s = t->stream;
  const Geo& G = t->g;
  DGeo g = dgeo(G);
  k_near<<<blocks_for(G.K, 128), 128, 0, s>>>(g, t->gsoff, t->gtoff, t->near, t->nnear, 0, G.K);
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  if (t->cfg.nranks <= 1) {
    t->leaf_lo = 0;
    t->leaf_hi = G.K;
    return FMM_OK;
  }
  int64_t nb = (G.K + FMM_PART_BLOCK - 1) / FMM_PART_BLOCK;
  double* bw = nullptr;
  FMM_CUDA_TRY(cudaMallocAsync((void**)&bw, nb * sizeof(double), s));
  k_block_work<<<(unsigned)nb, FMM_PART_BLOCK, 0, s>>>(G.K, t->gsoff, t->gtoff, t->near, t->nnear, G.p, bw);
  t->launches++;
  std::vector<double> hb(nb);
  cudaError_t ce = cudaMemcpyAsync(hb.data(), bw, nb * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  cudaFreeAsync(bw, s);
  FMM_CUDA_TRY(ce);
  return fmm_partition(hb.data(), nb, FMM_PART_BLOCK, G.K, t->cfg.rank, t->cfg.nranks, &t->leaf_lo, &t->leaf_hi);
}

int fmm_stage_tables_lists(fmm_tree_s* t) {
  cudaStream_t s = t->stream;
  const Geo& G = t->g;
  DGeo g = dgeo(G);
  LevelOffsets lvo;
  lvo.nl = G.L + 1;
  for (int l = 0; l <= G.L + 1; ++l) lvo.off[l] = G.lvl_off[l];
  k_centres<<<blocks_for(G.lvl_off[G.L + 1], 256), 256, 0, s>>>(g, lvo, t->centre);
  t->launches++;
  // single rank: near lists now (the multi-rank build made them before its local sort)
  if (t->cfg.nranks <= 1) {
    int e = fmm_stage_near_partition(t);
    if (e) return e;
  }
  // E4 candidates: source emptiness from the global counts, targets of this rank's range from
  // the local (kept) target CSR
  k_cand_level<<<blocks_for(G.lvl_off[G.L], 128), 128, 0, s>>>(g, lvo, t->gsoff, t->toff, t->cand, t->ncand,
                                                                t->leaf_lo, t->leaf_hi);
  k_e4mask_level<<<blocks_for(G.lvl_off[G.L + 1] - G.lvl_off[1], 128), 128, 0, s>>>(
      g, lvo, t->toff, t->cand, t->ncand, t->e4mask, t->leaf_lo, t->leaf_hi);
  t->launches += 2;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

namespace {
__global__ void k_gather_u(const int32_t* __restrict__ perm, int64_t n, const double* __restrict__ u,
                           double* __restrict__ su) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) su[i] = u[perm[i]];
}
}  // namespace

int fmm_stage_gather_strengths(fmm_tree_s* t, const double* u) {
  if (t->n_loc == 0) return FMM_OK;
  k_gather_u<<<blocks_for(t->n_loc, 256), 256, 0, t->stream>>>(t->sperm, t->n_loc, u, t->su);
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}
