// fmm_internal.cuh -- shared definitions of the B200 FMM library (CUDA, sm_100a).
// Product code only; never includes anything from oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/fmm_b200.h"

#define FMM_MAX_P 32
#define FMM_CAND_MAX 64  // >= 4*13 (triangle), 7*7 (septree), 4*9 (quad) E4 candidates per sibling group
#define FMM_NEAR_MAX 16  // >= 13 (triangle near set incl. self)
#define FMM_PART_BLOCK 32  // leaves per work block of the multi-rank partition (one warp)

// ---------------------------------------------------------------- host-side geometry constants
struct Geo {
  int tiling, L, B, p, self_mode;
  int nslot;              // max near-list length (partial-sum slots per target)
  int64_t K;              // B^L leaves
  int64_t ncells[17];     // B^l
  int64_t lvl_off[18];    // start of level l in the all-level cell arrays
  int64_t total_cells;
  double root_x, root_y, root_size;
  // septree: leaf circumradius and lattice factors (D8, D11)
  double sept_r, sept_A, sept_Bc, sept_D3r;
  int sept_K;             // |lattice coordinate| bound for in-domain points
};

// partial-sum slots per target of the near field: one per near leaf in self mode (symmetric
// blocks, p2p.cu), one in total for distinct targets (one task over all near leaves)
inline int fmm_part_slots(const Geo& g) { return g.self_mode ? g.nslot : 1; }

struct DevStatus {
  unsigned long long domain_bad;      // min offending index (ULLONG_MAX = none)
  unsigned long long coincident_bad;  // min offending target index
};

struct fmm_tree_s {
  fmm_config cfg;
  Geo g;
  cudaStream_t stream;
  int64_t n, m;
  int own_inputs;
  // inputs (device)
  const double* src_xy_in;  // interleaved
  const double* src_u_in;
  const double* tgt_xy_in;
  double* staging[3];       // device copies of host inputs (or NULL)
  // keys / permutation / CSR
  uint32_t* skey;  // [n]
  uint32_t* tkey;  // [m] (aliases skey in self mode)
  int32_t* sperm;  // [n] sorted position -> input index
  int32_t* tperm;  // [m]
  int32_t* soff;   // [K+2] leaf CSR of the sorted (rank-local) sources
  int32_t* toff;   // [K+2]
  // global leaf CSR (every rank's points; multi-rank: histogram + scan before the rank-local
  // sort; single rank: aliases soff / toff).  Emptiness tests of the lists and the work
  // estimate of the partition use these; data access uses the local soff / toff.
  int32_t* gsoff;  // [K+2]
  int32_t* gtoff;  // [K+2]
  int32_t* lflag;  // [K+1] multi-rank: bitmask ((K+32)/32 words, then K+1 byte flags) of the source leaves this rank
                   // keeps (own range U near halo)
  int64_t n_loc, m_loc;  // sorted (kept) sources / targets of this rank (= n, m on one rank)
  // sorted data
  double2* sxy;    // [n]
  double* su;      // [n]
  double2* txy;    // [m] (aliases sxy in self mode)
  // tree tables
  double2* centre; // [total_cells]
  int32_t* cand;   // [cells of levels 0..L-1][FMM_CAND_MAX]  E4 candidates of each parent, ascending
  int32_t* ncand;  // [cells of levels 0..L-1]
  unsigned long long* e4mask; // [total_cells] bit i <=> cand[parent][i] in E4(cell)
  int32_t* near;   // [K][FMM_NEAR_MAX]
  int32_t* nnear;  // [K]
  // P2P work list
  int4* tasks;         // [2 ntask_cap] per task (leaf t, q | q_rev << 8 | flags, row0, row1), (first target of t, first
                       // source / count of the columns, column leaf) of p2p.cu
  double2* part;       // [m][nslot] per (target, near-leaf) partial sums (Re, Im) of the near field
  int32_t* pskip;      // [K] per target leaf: bit q set <=> no task writes slot q (p2p.cu TF_PAIR)
  int32_t* ntask;      // [1] device counter
  int32_t* next_task;  // [1] dynamic scheduling counter of the P2P kernel
  int64_t ntask_cap;
  double* p2p_tab;     // [P2P_TAB_DOUBLES] log / atan tables of p2p_math.cuh
  // expansions
  double2* mp;     // [total_cells][p+1]
  double2* loc;    // [total_cells][p+1]
  double* binom;   // [(2P+1)][(2P+1)] binomial table
  double* afr;     // [FMM_AFR_MAX] the downward kernel's DMMA A fragments + 1/r table (fmm_down_afr_fill)
  // status
  DevStatus* status;
  // multi-rank leaf range and the multipole exchange
  int64_t leaf_lo, leaf_hi;
  fmm_comm_t comm;
  cudaStream_t xstream;   // high-priority side stream of the all-reduce (created on first use)
  cudaEvent_t xev[2];     // upward done (main -> side), all-reduce done (side -> main)
  int begun;              // fmm_evaluate_begin enqueued, fmm_evaluate_end pending
  // timing
  int timing, build_timed, eval_timed;
  cudaEvent_t ev[10];  // 0-7 stages (capi.cu); 8 keys done, 9 multi-rank selection done (build.cu)
  float stage_ms[6];
  int64_t launches;
  void* slab;  // single allocation holding every tree buffer
  size_t slab_bytes;
  int released;  // fmm_release: device buffers returned to the pool, timings kept
  // scratch for sort
  void* scratch;
  size_t scratch_bytes;
};

// ---------------------------------------------------------------- error helpers
void fmm_set_error_message(const std::string& s);
#define FMM_CUDA_TRY(expr)                                                                         \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess) {                                                                       \
      fmm_set_error_message(std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
      return _e == cudaErrorMemoryAllocation ? FMM_ENOMEM : FMM_ECUDA;                             \
    }                                                                                              \
  } while (0)

// ---------------------------------------------------------------- stage entry points (host)
// build.cu
int fmm_stage_keys_sort(fmm_tree_s* t);
int fmm_stage_near_partition(fmm_tree_s* t);
int fmm_stage_tables_lists(fmm_tree_s* t);
// comm.cu
int fmm_comm_allreduce_sum_f64(fmm_comm_t c, double* buf, size_t count, cudaStream_t s);
int32_t fmm_comm_nranks(fmm_comm_t c);
int32_t fmm_comm_rank(fmm_comm_t c);
int fmm_device_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* scratch, size_t scratch_bytes,
                        cudaStream_t s, int64_t* launches);
size_t fmm_scan_scratch_bytes(int64_t n);
int64_t fmm_scan_max_entries();  // largest input of fmm_device_scan_i32 (8192^2)
// the build's limits from its device scans (fmm_build_tree checks them up front): the K + 2 leaf
// counts and the radix digit histograms (1024 per 2048-point tile) must fit one scan
constexpr int64_t FMM_MAX_POINTS = (int64_t)1 << 27;
// passes.cu
// the downward kernel's per-order constants: the DMMA A fragments of the signed binomial matrix and
// the 1/r table, in the kernel's shared-memory layout, for template order P(p); binom = host table
constexpr int FMM_AFR_MAX = 4 * 8 * 32 + 8 * 4 + 8;
int fmm_down_order(int p);  // template order of p: 8, 12, ..., 32
int fmm_down_afr_fill(int P, const double* binom, double* out);  // returns the doubles written
int fmm_stage_upward(fmm_tree_s* t);
int fmm_stage_downward(fmm_tree_s* t);
int fmm_stage_p2p_pairs(fmm_tree_s* t);
int fmm_stage_p2p_finish(fmm_tree_s* t, double2* phi_out);
int fmm_build_tasks(fmm_tree_s* t);
bool fmm_p2p_pairing(const fmm_tree_s* t);  // p2p.cu: TF_PAIR tasks and the pairing kernel variant
int fmm_stage_gather_strengths(fmm_tree_s* t, const double* u);
int fmm_debug_p2p_math_launch(const double* dxdy, int64_t n, const double* tabs, double* out, cudaStream_t s);
// build.cu: the device geometry of a tree (geometry.cuh)
struct DGeo;
DGeo dgeo(const Geo& g);
// sample.cu (NEXT-4): leaf polygon of the regular-polygon point picking (D22):
// nsides, half-edge a, apothem b; apothem direction of edge z = (step z + off) pi / 6
struct SamplePoly {
  int nsides, step, off;
  double a, b;
};
int fmm_sample_launch(const Geo& G, const int64_t* cells, int64_t ncells, int per_cell, uint64_t seed, int64_t first,
                      const SamplePoly& P, double* xy, double* u, unsigned long long* bad, cudaStream_t s);
// capi.cu
void fmm_host_p2p_tables(double* tab);  // fills P2P_TAB_DOUBLES doubles
int fmm_direct_launch(const double* sxy, const double* su, int64_t n, const double* txy, int64_t m, int self_mode,
                      const double* tabs, double* phi, unsigned long long* bad, cudaStream_t s);
