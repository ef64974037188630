/*
 * fmm_oracle.h -- CPU ORACLE for the 2D log-kernel FMM of arXiv:1204.3105
 * (septree / triangle-quadtree / square quadtree).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product path (paper_1204_3105_b200/, include/fmm_b200.h) never includes,
 * links or calls anything here, and this file shares no code, header, table or
 * constant generator with it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation named);
 * D<k> = reading k in DESIGN.md "Readings of the paper" (ambiguities resolved).
 *
 * Parity pins: every function is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py against paper-printed values, closed forms,
 * invariants or brute force.  No function here
 * is "parity unpinned".
 */
#ifndef FMM_ORACLE_H
#define FMM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_QUAD = 0, ORC_SEPT = 1, ORC_TRIQ = 2 };

/* error codes */
enum { ORC_OK = 0, ORC_EBADCFG = 1, ORC_EDOMAIN = 2, ORC_ECOINCIDENT = 3, ORC_ENOMEM = 5 };

/* Frame of the root cell (D7, D8, D11):
 *   quad : root_x, root_y = lower-left corner of the root square, root_size = side
 *   sept : root_x, root_y = centre of leaf cell 0, root_size = R0 (idealised root
 *          hexagon circumradius); leaf circumradius r = R0 / (7^floor(L/2) * (L odd ? sqrt 7 : 1))
 *   triq : root_x, root_y = centroid of the upright root triangle, root_size = R0
 *          (root circumradius); level-l circumradius = ldexp(R0, -l)                    */
typedef struct {
  int32_t tiling;
  int32_t depth;      /* L = l_max >= 1 */
  int32_t p;          /* number of expansion terms (Q, a_1..a_p ; b_0..b_p) */
  int32_t self_mode;  /* targets == sources, pair (i,i) excluded by index (D16) */
  double root_x, root_y, root_size;
} orc_config;

/* ---- GBT arithmetic (septree). Digits are base-7, LSB first in
 *      arrays (d[0] = least significant = t_{|t|}). Returns result length. ---- */
int orc_gbt_add(const int32_t* a, int32_t la, const int32_t* b, int32_t lb, int32_t* out);
int orc_gbt_negate(const int32_t* a, int32_t la, int32_t* out);
int orc_gbt_zero_extend(int32_t j, int32_t m, int32_t* out);     /* eq. P:168 */
/* index helpers: base-7 integer <-> LSB-first digits */
int orc_gbt_index_add(int64_t a, int64_t b, int64_t* out);       /* a (*) b as base-7 integers */

/* ---- Tiling interface ---- */
int64_t orc_num_cells(const orc_config* c, int32_t level);           /* B^level */
/* Neighbors(n, l): fills out (<= 12 entries) in the paper's order, returns count */
int orc_neighbors(const orc_config* c, int32_t level, int64_t n, int64_t* out);
/* NeighborsE4(n, l): set difference reading (D1), all cells (no occupancy filter), sorted */
int orc_neighbors_e4(const orc_config* c, int32_t level, int64_t n, int64_t* out);
/* triangle adjacentNeighbor(n, k), k: 0 = L, 1 = R, 2 = V; -1 = none */
int64_t orc_triq_adjacent(int32_t level, int64_t n, int32_t k);
/* isUp(t, l) for an address t of |t| digits queried at level l */
int orc_triq_isup(int64_t t, int32_t ndigits, int32_t level);
/* CellCenter(n, l): exact-lattice form used for all FMM arithmetic (D12) */
void orc_cell_center(const orc_config* c, int32_t level, int64_t n, double* xy);
/* CellCenter(n, l) by the paper's polar formulas; cross-check only */
void orc_cell_center_polar(const orc_config* c, int32_t level, int64_t n, double* xy);
/* CellIndex(x, y, L) for every point: leaf keys; returns ORC_EDOMAIN and *bad = index */
int orc_keys(const orc_config* c, const double* xy, int64_t n, uint32_t* keys, int64_t* bad);
/* CellIndex at an arbitrary level (septree: prefix of the leaf address) */
int orc_cell_index(const orc_config* c, double x, double y, int32_t level, int64_t* out);

/* ---- Operators (classical GR forms, D10; P:43 omits them) ----
 * complex arrays are interleaved (re, im) doubles.  mp: [Q, a_1..a_p] (Q real stored
 * as complex), loc: [b_0..b_p]. centres are (x, y) pairs. */
void orc_p2m(const double* xy, const double* u, int64_t n, const double* c, int32_t p, double* mp);
void orc_m2m(const double* mp_child, const double* c_child, const double* c_parent, int32_t p, double* mp_parent_acc);
void orc_m2l(const double* mp, const double* c_m, const double* c_l, int32_t p, double* loc_acc);
void orc_l2l(const double* loc_parent, const double* c_parent, const double* c_child, int32_t p, double* loc_child_out);
void orc_l2p(const double* loc, const double* c, int32_t p, const double* y, double* phi);
/* Log(dx + i dy): principal branch, canonical +0 imaginary zero (D13) */
void orc_log(double dx, double dy, double* out);

/* ---- Direct summation, source-index order. tgt_ids: NULL = all targets ---- */
int orc_direct(const double* src_xy, const double* u, int64_t n, const double* tgt_xy, int64_t m,
               int32_t self_mode, const int64_t* tgt_ids, int64_t ntgt, double* phi, int64_t* bad);

/* ---- The FMM tree ---- */
typedef struct orc_tree orc_tree;
int orc_tree_build(const orc_config* c, const double* src_xy, const double* u, int64_t n,
                   const double* tgt_xy, int64_t m, orc_tree** out, int64_t* bad);
void orc_tree_free(orc_tree* t);
/* copies: keys of sources / targets (input order), sorted->original permutation */
void orc_tree_keys(const orc_tree* t, uint32_t* src_keys, uint32_t* tgt_keys);
void orc_tree_perm(const orc_tree* t, int32_t* src_perm, int32_t* tgt_perm);
void orc_tree_leaf_offsets(const orc_tree* t, int64_t* src_off, int64_t* tgt_off);
/* per-level occupancy */
int64_t orc_tree_count(const orc_tree* t, int32_t level, int64_t cell, int32_t which /*0 src 1 tgt*/);
/* interaction lists restricted to non-empty source cells, ascending (D17) */
int orc_tree_near(const orc_tree* t, int64_t leaf, int64_t* out);
int orc_tree_e4(const orc_tree* t, int32_t level, int64_t cell, int64_t* out);
/* the same lists as canonical CSR over the non-empty target cells (ascending):
 * owners [nown], offsets [nown+1], entries [nent].  Call with NULL buffers to get the
 * sizes in *nown / *nent. */
int orc_tree_near_csr(const orc_tree* t, int32_t* owners, int64_t* offs, int32_t* entries, int64_t* nown,
                      int64_t* nent);
int orc_tree_e4_csr(const orc_tree* t, int32_t level, int32_t* owners, int64_t* offs, int32_t* entries,
                    int64_t* nown, int64_t* nent);
/* CellCenter of every cell of a level (exact-lattice form, D12) */
void orc_tree_centres(orc_tree* t, int32_t level, double* xy);
/* upward pass over all cells (P2M + M2M) -- must be called before the getters below */
void orc_tree_upward(orc_tree* t);
void orc_tree_multipole(const orc_tree* t, int32_t level, int64_t cell, double* mp);
void orc_tree_multipoles_level(orc_tree* t, int32_t level, double* mp); /* all cells of a level */
/* local expansion of a target cell (computed on demand, level-ordered recursion) */
void orc_tree_local(orc_tree* t, int32_t level, int64_t cell, double* loc);
/* Phi at targets tgt_ids (original indices; NULL = all), returns ORC_ECOINCIDENT + *bad */
int orc_tree_evaluate(orc_tree* t, const int64_t* tgt_ids, int64_t ntgt, double* phi, int64_t* bad,
                      int64_t* counters /* [0] M2L ops, [1] P2P pairs, may be NULL */);
/* per-target accumulated paper bound B_j (D14) */
void orc_tree_bound(orc_tree* t, const int64_t* tgt_ids, int64_t ntgt, double* bound);

/* version / thread count used by OpenMP loops */
int orc_num_threads(void);
void orc_set_num_threads(int n);

/* NEXT-2: the appendix cost model and its depth of least cost (1..maxdepth) */
double orc_paper_cost(int tiling, double n, double m, int p, int depth);
int orc_paper_depth(int tiling, double n, double m, int p, int maxdepth);

/* NEXT-4: regular-polygon point picking in leaf cells (Fig. 12; reading D22).
 * Point g = first + i*per_cell + j (i < ncells, j < per_cell) is drawn uniformly in the leaf
 * polygon of cells[i] (cells == NULL: cell i) from the counter-based draws h(seed, 4g + d),
 * d = 0..3 (s, t, z, strength); xy[2(i*per_cell+j)..] = (x, y), u[...] = strength in [-1, 1)
 * (u may be NULL).  Returns ORC_EDOMAIN when a cell is outside [0, B^L). */
uint64_t orc_draw(uint64_t seed, uint64_t counter);
int orc_sample_cells(const orc_config* c, const int64_t* cells, int64_t ncells, int32_t per_cell, uint64_t seed,
                     int64_t first, double* xy, double* u);

#ifdef __cplusplus
}
#endif
#endif
