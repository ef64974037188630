/*
 * fmm_b200.h -- C ABI of the B200-native FMM hot path (libfmm_b200.so).
 *
 * Computes, for the complex log kernel of arXiv:1204.3105 section 2,
 *     Phi_j = sum_i u_i * Log(y_j - x_i),   j = 1..M           (eqs. 1-2)
 * by the hierarchical FMM on a fixed-depth square quadtree, septree (hexagons,
 * GBT addressing, section 5) or triangle-quadtree (section 6), with the
 * interaction lists of section 4 (Neighbors / NeighborsE4, read as a
 * set difference: DESIGN.md D1) and the classical 2D log-kernel operators the
 * paper cites but omits (D10).  Every step runs in this
 * library's own sm_100a CUDA kernels, in FP64.
 *
 * Plain C99: no C++ or torch types.  All functions are thread-compatible (one
 * tree per thread at a time).  Streams are passed as `void*` holding a
 * cudaStream_t (NULL = legacy default stream).
 *
 * Error codes (return values):
 *   FMM_OK            0
 *   FMM_EBADCFG       1  invalid configuration / argument
 *   FMM_EDOMAIN       2  a point lies outside the root domain (index: fmm_last_error_index)
 *   FMM_ECOINCIDENT   3  a target coincides with a source of another index (D16)
 *   FMM_ECUDA         4  CUDA runtime error (message: fmm_error_string / fmm_last_error_message)
 *   FMM_ENOMEM        5  device allocation failed
 *   FMM_ENCCL         6  NCCL unavailable or an NCCL call failed (message: fmm_last_error_message)
 *   FMM_EEXTENSION    7  the library was built without support for the request
 * Domain and coincidence errors are detected on the device; they are reported
 * by the next synchronising call (fmm_status, fmm_export).
 */
#ifndef FMM_B200_H
#define FMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMM_OK 0
#define FMM_EBADCFG 1
#define FMM_EDOMAIN 2
#define FMM_ECOINCIDENT 3
#define FMM_ECUDA 4
#define FMM_ENOMEM 5
#define FMM_ENCCL 6
#define FMM_EEXTENSION 7

/* tilings: square quadtree (Morton Z), septree, triangle-quadtree */
#define FMM_QUADTREE 0
#define FMM_SEPTREE 1
#define FMM_TRIQUAD 2

/* Multi-GPU communicator: an NCCL communicator owned by this
 * library (NCCL is loaded at run time from libnccl.so.2; no link-time dependency).  Rank 0
 * calls fmm_comm_unique_id and sends the FMM_COMM_ID_BYTES bytes to every rank (for example
 * by a torch.distributed broadcast); every rank then calls fmm_comm_init with its CUDA device
 * current.  One communicator serves any number of trees on that device, used from one host
 * thread at a time.  Errors: FMM_EBADCFG (arguments), FMM_ENCCL (NCCL missing or failing). */
#define FMM_COMM_ID_BYTES 128
typedef struct fmm_comm_s* fmm_comm_t;
int fmm_comm_unique_id(void* id);
int fmm_comm_init(const void* id, int32_t nranks, int32_t rank, fmm_comm_t* out);
int fmm_comm_destroy(fmm_comm_t comm);
/* NCCL version code of the loaded libnccl (e.g. 22809), 0 when NCCL cannot be loaded */
int fmm_nccl_version(void);

/* Configuration.  Frames (D7, D8, D11):
 *   FMM_QUADTREE: root_x, root_y = lower-left corner of the root square; root_size = its side.
 *   FMM_SEPTREE : root_x, root_y = centre of leaf cell 0 (origin of the leaf lattice);
 *                 root_size = R0, circumradius of the idealised root hexagon; the leaf
 *                 circumradius is r = R0 / (7^floor(L/2) * (L odd ? sqrt(7) : 1)); the domain
 *                 is the island of the 7^L leaf hexagons (reading D8).
 *   FMM_TRIQUAD : root_x, root_y = centroid of the upright root triangle; root_size = its
 *                 circumradius R0 (level-l circumradius R0 * 2^-l).
 * depth  L: quadtree / triangle 1..12, septree 1..9 for fmm_build_tree (the K + 2 leaf counts
 *           must fit one device scan of 8192^2 entries); the geometry-only calls
 *           (fmm_sample_cells) accept quadtree / triangle 1..15, septree 1..10 (32-bit keys).
 *           |root_x| + 2 root_size and |root_y| + 2 root_size must be < 1e20 (the P2P kernel
 *           pads with points at 1e30), root_size > 0, all finite; else FMM_EBADCFG.
 * p       : expansion terms, 1..31 (multipole Q, a_1..a_p; local b_0..b_p).
 * self_mode: 1 when targets are the sources; the pair (i, i) is skipped by index (D16).
 * rank / nranks: target-leaf partition for multi-GPU runs; single GPU: 0 / 1.
 *                Every rank gets the full input (replicated); it keys every point, cuts the
 *                leaves into work-balanced contiguous key ranges (fmm_partition; a range is a
 *                union of subtrees), and then sorts, keeps and evaluates only the
 *                points of its own leaf range plus the halo of near source leaves.  P2M / M2M
 *                run over its own source leaves only; the per-level multipole tree is summed
 *                over the ranks by one ncclAllReduce on `comm` (overlapped with the P2P pair
 *                kernel), or by the caller between fmm_evaluate_begin and fmm_evaluate_end.
 *                Rank r writes Phi of the targets in its leaf range only.
 * comm   : fmm_comm_t of this rank (nranks > 1), or NULL.  With nranks > 1 and comm NULL,
 *          fmm_evaluate is refused (FMM_EBADCFG); use the begin / end pair instead. */
typedef struct {
  int32_t tiling;
  int32_t depth;
  int32_t p;
  int32_t self_mode;
  double root_x;
  double root_y;
  double root_size;
  int32_t rank;
  int32_t nranks;
  int32_t flags;       /* FMM_FLAG_* */
  int32_t reserved[5]; /* must be zero */
  fmm_comm_t comm;     /* multi-GPU communicator or NULL */
} fmm_config;

/* flags: record per-stage CUDA events from fmm_build_tree on (see fmm_stage_times) */
#define FMM_FLAG_TIMING 1

typedef struct fmm_tree_s* fmm_tree_t;

/* Build the tree: leaf keys (CellIndex, P:207-250 / P:342-364 / Morton), a stable
 * sort of points by (leaf key, input index) -- a bucket sort for small leaves, else an LSD
 * radix sort --, leaf CSR offsets, cell centres (CellCenter, bit-exact
 * lattice form D12), the near / E4 interaction lists and the near-field task list.
 * n, m <= 2^27 and the depth limits of fmm_config, else FMM_EBADCFG with a message
 * (fmm_last_error_message).
 *
 * src_xy: n points as interleaved (x, y) float64 pairs (complex128 layout);
 * src_u : n real float64 strengths; tgt_xy: m points (ignored, may be NULL, in
 * self_mode where m must equal n).  Pointers may be device memory (used in
 * place) or host memory (copied to the device on `stream`; pinned memory makes
 * the copies asynchronous).  The library copies what it needs: inputs may be
 * freed or overwritten once the work on `stream` completes.
 * n == 0 or m == 0 is valid (potentials are then zero / empty).
 * Memory: the tree is one slab of the library's stream-ordered pool (fmm_tree_bytes; about
 * 0.65 KB per point in self mode at p = 24); during the build the sort takes scratch from the
 * same pool and returns it stream-ordered -- the bucket sort (K + 1) x 8 KB of leaf bins per
 * point set (it is only taken when that is <= 4 GB), the LSD sort about 40 B per point.
 * On success *out owns all device buffers until fmm_free. */
int fmm_build_tree(const fmm_config* cfg, const double* src_xy, const double* src_u, int64_t n,
                   const double* tgt_xy, int64_t m, void* stream, fmm_tree_t* out);

/* Evaluate Phi for all m targets of this rank: P2M, M2M (upward; multi-GPU: own leaves, then
 * the multipole all-reduce on a high-priority side stream), the P2P pair kernel, M2L + L2L per
 * level (downward), then the near-field sums and L2P.  phi_out: m complex128
 * values (interleaved re, im) in the caller's target order; device or host memory
 * (host: copied back on `stream`; the caller synchronises the stream).  Targets
 * owned by other ranks are left untouched.  Repeated evaluations are bitwise
 * identical unless the tree has heavy symmetric near blocks (self mode, two leaves
 * with n_t n_s > 65,536 points pairs), whose column sums are added atomically (equal
 * to rounding). */
int fmm_evaluate(fmm_tree_t t, double* phi_out, void* stream);

/* fmm_evaluate in two halves, for a multipole exchange done by the caller (nranks > 1 without
 * a comm; with a comm the all-reduce is enqueued by begin):
 *   begin: P2M + M2M over this rank's own source leaves (the partial multipole tree), then the
 *          P2P pair kernel (which needs no multipoles);
 *   end  : M2L + L2L over every level (using the multipole tree as it is in memory), the
 *          near-field sums and L2P into phi_out (as fmm_evaluate).
 * Between them the caller replaces the multipole tree (fmm_multipole_buffer) by the sum of
 * every rank's partial tree.  With nranks == 1 begin + end == fmm_evaluate. */
int fmm_evaluate_begin(fmm_tree_t t, void* stream);
int fmm_evaluate_end(fmm_tree_t t, double* phi_out, void* stream);
/* device pointer and byte size of the tree's multipole array: complex128 [cells of levels
 * 0..L][p+1], level-major (level l starts at cell sum_{k<l} B^k) */
int fmm_multipole_buffer(fmm_tree_t t, void** dev_ptr, size_t* bytes);

/* Replace the strengths (same geometry) so the tree can be re-evaluated. */
int fmm_set_strengths(fmm_tree_t t, const double* src_u, void* stream);

/* Synchronise the tree's stream and return the first device-detected error. */
int fmm_status(fmm_tree_t t);
/* offending input index of the last FMM_EDOMAIN (source index, or n + target index)
 * / FMM_ECOINCIDENT (target index); -1 if none */
int64_t fmm_last_error_index(fmm_tree_t t);

/* Exports for parity tests (synchronising, host buffers).  Returns the byte count
 * needed in *needed; copies min(bytes, needed) into host_buf when non-NULL.
 *   FMM_X_SRC_KEYS / FMM_X_TGT_KEYS : uint32 per input point (leaf index, input order)
 *   FMM_X_SRC_PERM / FMM_X_TGT_PERM : int32 per sorted position -> input index
 *   FMM_X_SRC_OFFSETS / FMM_X_TGT_OFFSETS : int64 [K+1] leaf CSR over the sorted order
 *   FMM_X_CENTRES  (level)  : float64 (x, y) per cell of the level, all B^level cells
 *   FMM_X_NEAR_OWNERS / _OFFSETS / _ENTRIES : near lists (D17) of the non-empty
 *                     target leaves: int32 owners ascending, int64 offsets, int32 entries
 *   FMM_X_E4_OWNERS / _OFFSETS / _ENTRIES (level) : NeighborsE4 lists likewise
 *   FMM_X_MULTIPOLE (level) : complex128 [B^level][p+1] (Q, a_1..a_p), after fmm_evaluate
 *   FMM_X_LOCAL     (level) : complex128 [B^level][p+1] (b_0..b_p) of evaluated cells
 *   FMM_X_COUNTERS : int64 [4] = {M2L ops, P2P pairs, non-empty source leaves, non-empty target leaves} */
#define FMM_X_SRC_KEYS 1
#define FMM_X_TGT_KEYS 2
#define FMM_X_SRC_PERM 3
#define FMM_X_TGT_PERM 4
#define FMM_X_SRC_OFFSETS 5
#define FMM_X_TGT_OFFSETS 6
#define FMM_X_CENTRES 7
#define FMM_X_NEAR_OWNERS 8
#define FMM_X_NEAR_OFFSETS 9
#define FMM_X_NEAR_ENTRIES 10
#define FMM_X_E4_OWNERS 11
#define FMM_X_E4_OFFSETS 12
#define FMM_X_E4_ENTRIES 13
#define FMM_X_MULTIPOLE 14
#define FMM_X_LOCAL 15
#define FMM_X_COUNTERS 16
int fmm_export(fmm_tree_t t, int32_t what, int32_t level, void* host_buf, size_t bytes, size_t* needed);

/* Per-stage device times (ms), from CUDA events on the tree's stream, of the build (when
 * cfg->flags has FMM_FLAG_TIMING) and of the last fmm_evaluate (when timing is on, by that
 * flag or fmm_set_timing(t, 1)): {keys + sort, centres + lists + tasks, P2P pair kernel,
 * P2M + M2M, M2L + L2L (all levels), P2P pair kernel + final sum/L2P}. */
int fmm_set_timing(fmm_tree_t t, int32_t enable);
int fmm_stage_times(fmm_tree_t t, float* ms6);
/* Build stage times (ms, FMM_FLAG_TIMING): {keying of every point, multi-rank selection (global
 * leaf counts, near lists, partition, halo, compaction; 0 on one rank), sort + gather of the
 * kept points, centres + E4 lists + P2P tasks}.  The first two are the work every rank repeats
 * on all points. */
int fmm_build_times(fmm_tree_t t, float* ms4);

/* Leaf range [lo, hi) of target leaves evaluated by cfg->rank (balanced by the
 * estimated near-field work; requires a built tree for the counts). */
int fmm_rank_range(fmm_tree_t t, int64_t* lo, int64_t* hi);

/* Work-balanced split of the target leaves for multi-GPU runs (host function; used by
 * fmm_build_tree when cfg->nranks > 1, exported for tests).  block_work[b] is the
 * estimated evaluation work of leaves [b*leaves_per_block, (b+1)*leaves_per_block);
 * rank r gets the leaf range [*lo, *hi) between the block boundaries whose prefix work
 * is closest to r*W/nranks and (r+1)*W/nranks.  Ranges of ranks 0..nranks-1 are
 * contiguous, disjoint and cover [0, K). */
int fmm_partition(const double* block_work, int64_t nblocks, int64_t leaves_per_block, int64_t K, int32_t rank,
                  int32_t nranks, int64_t* lo, int64_t* hi);

/* Grow the device's default stream-ordered memory pool by allocating and releasing
 * `bytes` (trees allocate from it; the library sets its release threshold to infinity). */
int fmm_pool_reserve(size_t bytes);
/* Device bytes held by a tree's slab. */
size_t fmm_tree_bytes(fmm_tree_t t);

/* Number of this library's kernel launches enqueued by the last build / evaluate. */
int64_t fmm_launch_count(fmm_tree_t t);

void fmm_free(fmm_tree_t t);

/* Return the tree's device buffers to the stream-ordered pool (freed on the tree's stream,
 * after the work already enqueued on it) while the handle stays valid for fmm_stage_times,
 * fmm_launch_count, fmm_rank_range and fmm_free.  Every call that needs device data
 * (fmm_evaluate, fmm_set_strengths, fmm_status, fmm_export) then returns FMM_EBADCFG.
 * Lets a caller run many build + evaluate steps back to back, reading the per-stage times
 * afterwards, with the memory of one step live at a time.  Errors: FMM_EBADCFG (NULL). */
int fmm_release(fmm_tree_t t);

/* Depth selection.  Cost of one build + evaluate at `depth`:
 *   uc == NULL: the paper's appendix model (Table 2),
 *     (M+N) p + K B/(B-1) (P4+2) p^2 + M (P2 N/K + p),  K = B^depth  (constant term dropped);
 *   uc != NULL: a device-time model in the units of uc,
 *     c0 + c_point (N+M)(p+1) + c_cell K B/(B-1) (P4+2) (p+1)^2 + c_pair M P2 N/K + c_leaf K,
 * with (B, P4, P2) = (4, 27, 9) quadtree, (7, 42, 7) septree, (4, 39, 13) triangle-quadtree.
 * fmm_choose_depth returns the depth of least cost (first minimum) in 1..10 (septree) or 1..15.
 * Host only (no device work).  Errors: FMM_EBADCFG. */
typedef struct {
  double c0, c_point, c_cell, c_pair, c_leaf;
} fmm_unit_costs;
int fmm_predict_cost(int32_t tiling, int64_t n, int64_t m, int32_t p, int32_t depth, const fmm_unit_costs* uc,
                     double* cost);
int fmm_choose_depth(int32_t tiling, int64_t n, int64_t m, int32_t p, const fmm_unit_costs* uc, int32_t* depth);

/* Direct evaluation (the reference of the paper's section-9 error and
 * runtime sweeps): phi_out[j] = sum_i src_u[i] Log(tgt_j - src_i) over all n
 * sources, O(n m), principal branch with a canonical +0 imaginary zero (D13); in self_mode
 * (targets = sources, m == n, tgt_xy ignored) the pair i == j is skipped (D16).  Pointers as
 * in fmm_build_tree (device used in place, host staged on `stream`); phi_out m complex128 on
 * the device or host.  Synchronises `stream`.  Returns FMM_ECOINCIDENT (message names the
 * smallest target index) when a target coincides with a source of another index. */
int fmm_direct(const double* src_xy, const double* src_u, int64_t n, const double* tgt_xy, int64_t m,
               int32_t self_mode, double* phi_out, void* stream);

/* Device-side input generation: regular-polygon point picking in
 * leaf cells, PAPER.md P:426-433 and Fig. 12 -- the leaf polygon is cut into one isosceles
 * triangle per edge, halves of each triangle are rearranged into an a x b rectangle
 * (half-edge x apothem), (s, t) is uniform in the rectangle and z uniform in the edges.
 * Leaf polygons: square of side root_size 2^-L; hexagon of circumradius r (D8) with a vertex
 * at angle 0; triangle of circumradius root_size 2^-L, upright or inverted (isUp);
 * centred at CellCenter of the leaf (D12).
 *
 * Point o (0 <= o < ncells * per_cell) lies in leaf cells[o / per_cell] (cells == NULL: leaf
 * o / per_cell, ncells <= B^L) and is point g = first + o of the sample: its draws are the
 * counter-based SplitMix64 outputs h(seed, 4g + d), d = 0..3 (reading D22), so that a rank
 * or a check can generate any slice alone.  xy: device, interleaved (x, y) float64 pairs,
 * ncells * per_cell of them; u: device strengths 2 h_3 2^-53 - 1 in [-1, 1), or NULL;
 * cells: device int64 or NULL.  Bit-identical to the oracle's sampler (every rounding fixed).
 * Synchronises `stream`.  Errors: FMM_EBADCFG (config, sizes, host pointers),
 * FMM_EDOMAIN (a cell outside [0, B^L); message names the smallest cells index). */
int fmm_sample_cells(const fmm_config* cfg, const int64_t* cells, int64_t ncells, int32_t per_cell, uint64_t seed,
                     int64_t first, double* xy, double* u, void* stream);

/* Test hook: the P2P kernel's FP64 math on n explicit offsets z = dx + i dy (device
 * pointers, interleaved): out[2i] = log|z|^2, out[2i+1] = Arg z in (-pi, pi] with a zero
 * imaginary part read as +0 (D13).  z must have a normal |z|^2 (the kernel
 * sends zero / subnormal |z|^2 to an exact slow path).  Synchronises `stream`. */
int fmm_debug_p2p_math(const double* dxdy, int64_t n, double* out, void* stream);
const char* fmm_error_string(int code);
const char* fmm_last_error_message(void);
int fmm_version(void);

#ifdef __cplusplus
}
#endif
#endif
