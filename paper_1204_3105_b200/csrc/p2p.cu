// p2p.cu -- the near field, Phi_near(y_j) = sum over near leaves of sum_i u_i Log(y_j - x_i)
// (SURVEY §8(a) a11), fused with L2P of the leaf locals and the
// store at the caller's index (a10, a12).
//
// Work unit = one (target leaf t, near leaf s) block.  In self mode (targets = sources,
// reading D16) the near relation is symmetric, and so is the kernel up to the branch of
// Arg: Log(x_i - x_j) = Log(x_j - x_i) +/- i pi, with the same log|z|^2.  An off-diagonal
// block (t < s) is therefore evaluated ONCE: every pair feeds the row target
// (u_j Log(x_i - x_j)) and, reversed, the column target (u_i Log(x_j - x_i)).  Light blocks
// (n_t n_s <= 65,536) are one task; heavy ones are split by rows of the larger leaf.
// Diagonal blocks are symmetric as well (schedule below; heavy ones split by rows).  Every
// (target, near-leaf) pair of the near list owns one partial-sum slot, and a final pass adds
// the slots in near-list order.  Each slot is written by exactly one task, so the result is
// bitwise reproducible, except the slots of heavy symmetric blocks, which several row-range
// tasks add into atomically.  Distinct targets (one-sided) take one task per target leaf over
// the sources of all its near leaves, concatenated in near-list order, and one slot per target.
#include <type_traits>

#include "fmm_internal.cuh"
#include "p2p_math.cuh"

namespace {

constexpr int P2P_LIGHT = 1 << 16;  // max pairs of one symmetric (single-warp) block
constexpr int P2P_S = 192;          // sources of one near leaf kept in shared memory per warp
constexpr int P2P_SD = 320;         // distinct targets: near-list sources kept in shared memory per warp
constexpr int TF_SYM = 1 << 16, TF_DIAG = 1 << 17, TF_HEAVY = 1 << 18;
// TF_PAIR (self mode): two light off-diagonal blocks (t, s1), (t, s2) of one row leaf in one task,
// the columns s1's sources then s2's (<= P2P_S together, staged once):
// y = q1 | q1r << 8 | flags | q2 << 20 | q2r << 24 (FMM_NEAR_MAX = 16); the row sums go to slot q1,
// slot q2 of the rows is never written and the finish skips it (pskip).  Only the staging and the
// task's last writes read the pair fields.
constexpr int TF_PAIR = 1 << 19;

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// rows per one-sided task of a block with ns sources (a multiple of 8, >= 8)
__device__ __forceinline__ int split_rows(int ns) { return max(8, (P2P_LIGHT / max(ns, 1)) & ~7); }

// tasks of target leaf t: count (out == nullptr) or write them from *pos
// mode: bit 0 = self mode, bit 1 = TF_PAIR tasks allowed (the pairing kernel variant runs)
// skip (optional): the slots of t's targets no task writes (slot q2 of every TF_PAIR task)
__device__ int leaf_tasks(int t, const int32_t* __restrict__ toff, const int32_t* __restrict__ soff,
                          const int32_t* __restrict__ near, const int32_t* __restrict__ nnear, int mode,
                          int64_t lo, int64_t hi, int4* out, int32_t* skip = nullptr) {
  if (skip) *skip = 0;
  const int nt = toff[t + 1] - toff[t];
  if (nt == 0) return 0;
  const bool self_mode = mode & 1, pairs = (mode >> 1) & 1;
  const bool t_in = t >= lo && t < hi;
  const int nn = nnear[t];
  int c = 0;
  // a task is two int4: (row leaf, slot | reverse slot << 8 | flags, row range) and the values the
  // pair kernel would otherwise load one after another (first sorted target of the row leaf,
  // first source and source count of the column leaf -- all near leaves for distinct targets --,
  // column leaf)
  auto put = [&](int4 a, int ncols) {
    if (out) {
      const int s = near[(int64_t)a.x * FMM_NEAR_MAX + (a.y & 0xff)];
      out[2 * c] = a;
      out[2 * c + 1] = make_int4(toff[a.x], soff[s], ncols, s);
    }
    ++c;
  };
  auto put_pair = [&](int q1, int q1r, int q2, int q2r) {
    if (out) {
      out[2 * c] = make_int4(t, q1 | (q1r << 8) | TF_SYM | TF_PAIR | (q2 << 20) | (q2r << 24), 0, nt);
      out[2 * c + 1] = make_int4(0, 0, 0, 0);
    }
    if (skip) *skip |= 1 << q2;
    ++c;
  };
  auto emit_rows = [&](int leaf, int qq, int rows, int ns, int flags) {
    const int rs = split_rows(ns);
    for (int r0 = 0; r0 < rows; r0 += rs) put(make_int4(leaf, qq | flags, r0, min(rows, r0 + rs)), ns);
  };
  if (!self_mode) {
    // distinct targets: one task (row ranges of <= 65,536 pairs) over ALL near leaves of t, their
    // sources concatenated in near-list order as the columns; one partial-sum slot per target
    if (!t_in) return 0;
    int tot = 0;
    for (int q = 0; q < nn; ++q) {
      const int s = near[(int64_t)t * FMM_NEAR_MAX + q];
      tot += soff[s + 1] - soff[s];
    }
    if (tot > 0) emit_rows(t, 0, nt, tot, 0);
    return c;
  }
  // a light block of an own row leaf waiting for a partner (TF_PAIR): slot, reverse slot, sources
  int pq = -1, pqr = 0, pns = 0;
  for (int q = 0; q < nn; ++q) {
    const int s = near[(int64_t)t * FMM_NEAR_MAX + q];
    const int ns = soff[s + 1] - soff[s];
    if (s < t) continue;  // the block belongs to the smaller leaf index
    if (s == t) {  // diagonal block: symmetric (each unordered pair once) when it fits a warp
      if (t_in) {
        if (ns <= P2P_S) {
          put(make_int4(t, q | (q << 8) | TF_SYM | TF_DIAG, 0, nt), ns);
        } else {
          // heavy diagonal: symmetric row ranges; rows and reactions meet in slot q and are
          // added atomically (zeroed by k_heavy_zero)
          emit_rows(t, q | (q << 8), nt, ns, TF_SYM | TF_DIAG | TF_HEAVY);
        }
      }
      continue;
    }
    const bool s_in = s >= lo && s < hi;
    // index of t in near(s)
    int qr = 0;
    for (int k = 0; k < nnear[s]; ++k)
      if (near[(int64_t)s * FMM_NEAR_MAX + k] == t) qr = k;
    if ((int64_t)nt * ns <= P2P_LIGHT) {
      if (pairs && t_in && ns <= P2P_S) {
        // paired with the previous light block of t when both column leaves fit shared memory
        if (pq >= 0 && pns + ns <= P2P_S) {
          put_pair(pq, pqr, q, qr);
          pq = -1;
        } else {
          if (pq >= 0) put(make_int4(t, pq | (pqr << 8) | TF_SYM, 0, nt), pns);
          pq = q;
          pqr = qr;
          pns = ns;
        }
      } else if (t_in || s_in) {
        put(make_int4(t, q | (qr << 8) | TF_SYM, 0, nt), ns);
      }
    } else if (t_in || s_in) {
      // heavy block: symmetric too, split by rows of the larger leaf; the smaller one is the
      // column side (kept in shared memory when it fits) whose reactions from the row ranges
      // are added atomically (their order is not fixed: reading D15's tolerance, not bits)
      const bool t_rows = nt >= ns;
      emit_rows(t_rows ? t : s, t_rows ? (q | (qr << 8)) : (qr | (q << 8)), t_rows ? nt : ns, t_rows ? ns : nt,
                TF_SYM | TF_HEAVY);
    }
  }
  if (pq >= 0) put(make_int4(t, pq | (pqr << 8) | TF_SYM, 0, nt), pns);
  return c;
}

// zero the column-side slots of every heavy symmetric block (once per block: its r0 = 0 task)
__global__ void k_heavy_zero(const int4* __restrict__ tasks, const int32_t* __restrict__ ntask_p,
                             const int32_t* __restrict__ soff, const int32_t* __restrict__ near,
                             double2* __restrict__ part, int nslot) {
  const int ntask = *ntask_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ntask; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 tk = tasks[2 * i];
    if (!(tk.y & TF_HEAVY) || tk.z != 0) continue;
    const int s = tasks[2 * i + 1].w, qr = (tk.y >> 8) & 0xff;
    for (int j = soff[s]; j < soff[s + 1]; ++j) part[(int64_t)j * nslot + qr] = make_double2(0.0, 0.0);
  }
}

__global__ void k_task_count(int64_t K, const int32_t* __restrict__ toff, const int32_t* __restrict__ soff,
                             const int32_t* __restrict__ near, const int32_t* __restrict__ nnear, int self_mode,
                             int64_t lo, int64_t hi, int32_t* __restrict__ cnt) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > K) return;
  cnt[t] = t < K ? leaf_tasks((int)t, toff, soff, near, nnear, self_mode, lo, hi, nullptr) : 0;
}

__global__ void k_task_fill(int64_t K, const int32_t* __restrict__ toff, const int32_t* __restrict__ soff,
                            const int32_t* __restrict__ near, const int32_t* __restrict__ nnear, int self_mode,
                            int64_t lo, int64_t hi, const int32_t* __restrict__ start, int4* __restrict__ tasks,
                            int32_t* __restrict__ ntask, int32_t* __restrict__ pskip) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > K) return;
  if (t == K) {
    *ntask = start[K];
    return;
  }
  leaf_tasks((int)t, toff, soff, near, nnear, self_mode, lo, hi, tasks + 2 * (int64_t)start[t], pskip + t);
}

// ------------------------------------------------------------------ the pair kernel
// Lane = (row lane tl = lane % 4, phase ph = lane / 4).  A row step covers 8 target rows: the
// lane owns rows tl and tl + 4.  Sources of s are staged 32 at a time in shared memory and a
// lane visits columns 16 h + 8 j + ph (h, j in {0, 1}): 2 rows x 2 columns per (h) step.
// Padding replaces every validity test in the pair loop: missing rows sit at (PAD, PAD) with
// u = 0, missing columns at (-PAD, PAD) with u = 0 (coordinates are < 1e20 in magnitude,
// make_geo), so their terms are exactly 0 and no pair of them is near.  The excluded pair
// (i, i) of a diagonal block (D16) is the only z = 0 that is not an error.
#ifndef P2P_WARPS
#define P2P_WARPS 16  // warps per block (the tables are shared by the block; 16 x 1 block beat 8 x 2 by 0.25 %)
#endif
#ifndef P2P_MINB
#define P2P_MINB 1  // resident blocks per SM the register allocation is sized for (16 warps: 128 registers)
#endif
constexpr int P2P_RS = 32;  // row stride (double2) of the reaction scratch; column c of row lane r sits at c ^ 2r
                            // (conflict-free STS.128 / LDS.128)
// dynamic shared memory of one block: tables, then per warp sources, strengths, reactions, scratch
constexpr size_t P2P_TAB_BYTES = sizeof(double2) * (P2P_LOG_N + P2P_ATAN_N);
constexpr size_t P2P_WARP_BYTES = sizeof(double2) * (2 * P2P_S + 4 * P2P_RS) + sizeof(double) * P2P_S;
constexpr size_t P2P_SMEM = P2P_TAB_BYTES + P2P_WARPS * P2P_WARP_BYTES;
static_assert(24 * P2P_SD + 64 * sizeof(double2) <= P2P_WARP_BYTES, "distinct-target warp layout");
constexpr double P2P_PAD = 1.0e30;

struct PairOut {
  double lg, ag;  // log|z|^2, Arg z
};

// log|z|^2 and Arg z of z = dx + i dy for |z| >= 1e-30 (branch-free, so that the compiler
// overlaps the pairs of a column).  Smaller |z| give finite table indices (s_atan is padded)
// and garbage values, which p2p_slow replaces.
__device__ __forceinline__ PairOut p2p_fast(double dx, double dy, double r2, uint32_t s_log, uint32_t s_atan) {
  PairOut o;
  double kd, lz;
  p2p_log_split(r2, s_log, &kd, &lz);
  o.lg = fma(kd, P2P_C[12], lz);  // kd ln 2 + lz (one rounding of the exact product sum)
  o.ag = p2p_atan2<true>(dy, dx, s_atan);
  return o;
}

// |z| < 1e-30: exact libdevice path; z = 0 is the excluded pair (i, i) of a diagonal block
// (D16) or coincident points (an error: the smallest caller index involved is reported)
__device__ __noinline__ PairOut p2p_slow(double dx, double dy, double r2, bool self_ok, const int32_t* tperm,
                                         int trow, int scol, DevStatus* st) {
  PairOut o;
  if (r2 == 0.0) {
    if (!self_ok) {
      unsigned long long bad = (unsigned long long)tperm[trow];
      if (scol >= 0) bad = min(bad, (unsigned long long)tperm[scol]);
      atomicMin(&st->coincident_bad, bad);
    }
    o.lg = 0.0;
    o.ag = 0.0;
  } else {
    o.lg = 2.0 * log(hypot(dx, dy));
    o.ag = atan2(__dadd_rn(dy, 0.0), dx);  // D13
  }
  return o;
}

// TF_PAIR staging: s1's sources [sb, sb + n1) then s2's into s_xy / s_u (padded to a multiple of
// 32), reactions zeroed; returns the column count.
__device__ __forceinline__ int p2p_stage_pair(int ty, int t, int sb, int n1, const int32_t* __restrict__ soff,
                                              const int32_t* __restrict__ near, const double2* __restrict__ sxy,
                                              const double* __restrict__ su, double2* s_xy, double* s_u,
                                              double2* s_re) {
  const int lane = threadIdx.x & 31;
  const int s2 = near[(int64_t)t * FMM_NEAR_MAX + ((ty >> 20) & 15)];
  const int sb2 = soff[s2], ns = n1 + soff[s2 + 1] - sb2;
  for (int i = lane; i < ((ns + 31) & ~31); i += 32) {
    if (i < ns) {
      const int j = i < n1 ? sb + i : sb2 + (i - n1);
      s_xy[i] = sxy[j];
      s_u[i] = su[j];
    } else {
      s_xy[i] = make_double2(-P2P_PAD, P2P_PAD);
      s_u[i] = 0.0;
    }
    s_re[i] = make_double2(0.0, 0.0);
  }
  __syncwarp();
  return ns;
}

// TF_PAIR last writes: the two column leaves' reactions to their reverse slots (slot q2 of the rows
// stays unwritten: the finish skips it, pskip)
__device__ __forceinline__ void p2p_finish_pair(int ty, int t, int tb, int nrows, int sb, int qr, int ns,
                                                bool write_rows, bool write_react, int64_t lo, int64_t hi,
                                                const int32_t* __restrict__ soff, const int32_t* __restrict__ near,
                                                const double2* s_re, double2* __restrict__ part, int nslot) {
  const int lane = threadIdx.x & 31;
  const int s1 = near[(int64_t)t * FMM_NEAR_MAX + (ty & 0xff)];
  const int n1 = soff[s1 + 1] - soff[s1], q2 = (ty >> 20) & 15, q2r = (ty >> 24) & 15;
  const int s2 = near[(int64_t)t * FMM_NEAR_MAX + q2], sb2 = soff[s2];
  const bool write_react2 = s2 >= lo && s2 < hi;
  for (int i = lane; i < ns; i += 32) {
    if (i < n1) {
      if (write_react) part[(int64_t)(sb + i) * nslot + qr] = s_re[i];
    } else if (write_react2) {
      part[(int64_t)(sb2 + i - n1) * nslot + q2r] = s_re[i];
    }
  }
  (void)write_rows;
  (void)tb;
  (void)nrows;
}

// SELF: self mode (symmetric tasks possible); the distinct-target instantiation has no
// reversed-pair work at all
// PAIRS: the variant that runs TF_PAIR tasks (self mode; fmm_p2p_pairing decides)
template <bool SELF, bool PAIRS>
__global__ void __launch_bounds__(32 * P2P_WARPS, P2P_MINB) k_p2p_pairs(
    const int4* __restrict__ tasks, const int32_t* __restrict__ ntask_p, int32_t* __restrict__ next_task,
    const int32_t* __restrict__ toff, const int32_t* __restrict__ soff, const double2* __restrict__ txy,
    const double2* __restrict__ sxy, const double* __restrict__ su, const int32_t* __restrict__ near,
    const int32_t* __restrict__ nnear, const int32_t* __restrict__ tperm, const double* __restrict__ tabs,
    double2* __restrict__ part, int nslot, int64_t lo, int64_t hi, DevStatus* st) {
  extern __shared__ double2 smem[];
  double2* s_log = smem;
  double2* s_atan = s_log + P2P_LOG_N;  // P2P_ATAN_N entries (garbage k of |z| < 1e-30 stays inside)
  p2p_load_tables(tabs, s_log, s_atan);
  const uint32_t a_log = p2p_smem_addr(s_log), a_atan = p2p_smem_addr(s_atan);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* const s_xy = (double2*)((char*)smem + P2P_TAB_BYTES + w * P2P_WARP_BYTES);  // sources of s
  // self mode: s_xy[P2P_S], reactions s_re[P2P_S], scratch s_rs[4 P2P_RS], strengths s_u[P2P_S];
  // distinct targets (no reactions): s_xy[P2P_SD], s_u[P2P_SD], row-sum scratch s_rs[64]
  double2* const s_re = s_xy + P2P_S;    // reactions of the sources of s (self mode)
  double2* const s_rs = SELF ? s_re + P2P_S : (double2*)((char*)s_xy + 24 * P2P_SD);
  double* const s_u = SELF ? (double*)(s_rs + 4 * P2P_RS) : (double*)(s_xy + P2P_SD);
  const int tl = lane & 3, ph = lane >> 2;
  const double PI = 3.141592653589793;
  const int ntask = *ntask_p;
  while (true) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= ntask) break;
    const int4 tk = tasks[2 * task];
    const int t = tk.x, q = tk.y & 0xff, qr = (tk.y >> 8) & 0xff;
    const bool sym = SELF && (tk.y & TF_SYM), diag = SELF && (tk.y & TF_DIAG), heavy = SELF && (tk.y & TF_HEAVY);
    // symmetric diagonal block: a row step of rows [rc, rc + 8) and a 16-column half at a
    // skips the half when a + 15 < rc (those pairs arrive as reactions of earlier row steps),
    // evaluates it one-sided when it straddles the rows (a <= rc + 7; the pair (i, i) is the
    // excluded z = 0) and symmetrically when it lies above them; each ordered pair i != j
    // is then counted once (tests/test_p2p_schedule.py enumerates the rule)
    const bool sd = sym && diag;
    // distinct targets: first target of t, count of the concatenated columns from the task's
    // second half (one memory round trip); self mode: loaded here, which keeps the symmetric
    // kernel's register allocation (holding the second half through the pair loop cost it 1.5 %)
    int tb, sb, ns, s;
    if (SELF) {
      s = near[(int64_t)t * FMM_NEAR_MAX + q];
      tb = toff[t];
      sb = soff[s];
      ns = soff[s + 1] - sb;
    } else {
      const int4 tx = tasks[2 * task + 1];
      tb = tx.x;
      sb = tx.y;
      ns = tx.z;
      s = tx.w;
    }
    // distinct targets: the columns are the sources of all near leaves of t, concatenated
    const int nn = SELF ? 1 : nnear[t];
    // sorted position of column c of the concatenation (distinct targets, c < ns)
    auto col_src = [&](int c) -> int {
      if (SELF) return sb + c;
      for (int k = 0;; ++k) {
        const int s2 = near[(int64_t)t * FMM_NEAR_MAX + k];
        const int b2 = soff[s2], n2 = soff[s2 + 1] - b2;
        if (c < n2) return b2 + c;
        c -= n2;
      }
    };
    const bool write_rows = t >= lo && t < hi;
    const bool write_react = sym && s >= lo && s < hi;
    // ns <= P2P_S (P2P_SD): the sources (padded to a multiple of 32) stay in shared memory for
    // the task and the reactions accumulate there; larger leaves are restaged per row step and chunk
    const bool whole = ns <= (SELF ? P2P_S : P2P_SD);
    if (whole && !SELF) {
      int off = 0;
      for (int k = 0; k < nn; ++k) {
        const int s2 = near[(int64_t)t * FMM_NEAR_MAX + k];
        const int b2 = soff[s2], n2 = soff[s2 + 1] - b2;
        for (int i = lane; i < n2; i += 32) {
          s_xy[off + i] = sxy[b2 + i];
          s_u[off + i] = su[b2 + i];
        }
        off += n2;
      }
      for (int i = ns + lane; i < ((ns + 31) & ~31); i += 32) {
        s_xy[i] = make_double2(-P2P_PAD, P2P_PAD);
        s_u[i] = 0.0;
      }
      __syncwarp();
    } else if (PAIRS && (tk.y & TF_PAIR)) {
      ns = p2p_stage_pair(tk.y, t, sb, ns, soff, near, sxy, su, s_xy, s_u, s_re);
    } else if (whole) {
      for (int i = lane; i < ((ns + 31) & ~31); i += 32) {
        if (i < ns) {
          s_xy[i] = sxy[sb + i];
          s_u[i] = su[sb + i];
        } else {
          s_xy[i] = make_double2(-P2P_PAD, P2P_PAD);
          s_u[i] = 0.0;
        }
        s_re[i] = make_double2(0.0, 0.0);
      }
      __syncwarp();
    }
    for (int rc = tk.z; rc < tk.w; rc += 8) {
      const int row0 = rc + tl, row1 = row0 + 4;
      const bool v0 = row0 < tk.w, v1 = row1 < tk.w;
      const double2 y0 = v0 ? txy[tb + row0] : make_double2(P2P_PAD, P2P_PAD);
      const double2 y1 = v1 ? txy[tb + row1] : make_double2(P2P_PAD, P2P_PAD);
      // self mode: the row targets are also sources (their strengths weight the reactions)
      const double u0 = (sym && v0) ? su[tb + row0] : 0.0, u1 = (sym && v1) ? su[tb + row1] : 0.0;
      double a0r = 0.0, a0i = 0.0, a1r = 0.0, a1i = 0.0;
      // a last row step of <= 4 rows: distinct targets and the pairing variant (non-diagonal
      // tasks); in the plain symmetric kernel the extra path costs the main loop more (register
      // allocation) than the empty rows it saves, in the pairing variant it saves 1.2-1.4 %
      const bool last4 = (!SELF || (PAIRS && !sd)) && tk.w - rc <= 4;
      for (int c0 = sd ? (rc & ~31) : 0; c0 < ns; c0 += 32) {
        if (!whole) {
          if (c0 + lane < ns) {
            const int i = col_src(c0 + lane);
            s_xy[lane] = sxy[i];
            s_u[lane] = su[i];
          } else {
            s_xy[lane] = make_double2(-P2P_PAD, P2P_PAD);
            s_u[lane] = 0.0;
          }
          __syncwarp();
        }
        const int cb = whole ? c0 : 0;  // chunk base in shared memory
        const int cnt = min(32, ns - c0);
        unsigned hw = 0;  // halves of the chunk whose reaction partials are in s_rs
        if (last4) {
          // a last row step of <= 4 rows: one row (tl) and 4 columns 8 j + ph of the chunk per
          // lane, so that the empty rows tl + 4 cost nothing
          double vr[4] = {0.0, 0.0, 0.0, 0.0}, vi[4] = {0.0, 0.0, 0.0, 0.0};
          auto cols1 = [&](auto njc) {
            constexpr int NJ = decltype(njc)::value;
            double uc[NJ], dx[NJ], dy[NJ], r2[NJ];
            PairOut pr[NJ];
            bool slow = false;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              const double2 x = s_xy[cb + 8 * j + ph];
              uc[j] = s_u[cb + 8 * j + ph];
              dx[j] = y0.x - x.x;
              dy[j] = y0.y - x.y;
              r2[j] = fma(dx[j], dx[j], dy[j] * dy[j]);
              pr[j] = p2p_fast(dx[j], dy[j], r2[j], a_log, a_atan);
              slow |= __double2hiint(r2[j]) < P2P_SLOW_HI;
            }
            if (__builtin_expect(slow, 0)) {
#pragma unroll
              for (int j = 0; j < NJ; ++j) {
                const int col = c0 + 8 * j + ph;
                if (__double2hiint(r2[j]) < P2P_SLOW_HI)
                  pr[j] = p2p_slow(dx[j], dy[j], r2[j], false, tperm, tb + row0, sym ? sb + col : -1, st);
              }
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              a0r = fma(uc[j], pr[j].lg, a0r);
              a0i = fma(uc[j], pr[j].ag, a0i);
              const double g = pr[j].ag;
              vr[j] = u0 * pr[j].lg;
              vi[j] = u0 * (g > 0.0 ? g - PI : g + PI);
            }
          };
          if (cnt > 16)
            cols1(std::integral_constant<int, 4>{});
          else
            cols1(std::integral_constant<int, 2>{});
          if (sym) {
#pragma unroll
            for (int j = 0; j < 4; ++j) s_rs[tl * P2P_RS + ((8 * j + ph) ^ (2 * tl))] = make_double2(vr[j], vi[j]);
            hw = cnt > 16 ? 3u : 1u;
          }
        } else
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && cnt <= 16) break;  // a short last chunk skips its empty second half
          const int a = c0 + 16 * h;
          if (sd && a + 15 < rc) continue;
          const bool react = sym && !(sd && a <= rc + 7);
          const bool two = cnt - 16 * h > 8;  // ... and an empty last quarter
          double vr[2] = {0.0, 0.0}, vi[2] = {0.0, 0.0};
          // NJ columns x 2 rows in one basic block (the slow-path test covers all of them), so
          // that the compiler overlaps the 2 NJ independent pairs
          auto cols = [&](auto njc) {
            constexpr int NJ = decltype(njc)::value;
            double2 x[NJ];
            double uc[NJ], dx[NJ][2], dy[NJ][2], r2[NJ][2];
            PairOut pr[NJ][2];
            bool slow = false;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              const int k = 16 * h + 8 * j + ph;
              x[j] = s_xy[cb + k];
              uc[j] = s_u[cb + k];
              dx[j][0] = y0.x - x[j].x;
              dy[j][0] = y0.y - x[j].y;
              dx[j][1] = y1.x - x[j].x;
              dy[j][1] = y1.y - x[j].y;
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                r2[j][r] = fma(dx[j][r], dx[j][r], dy[j][r] * dy[j][r]);
                pr[j][r] = p2p_fast(dx[j][r], dy[j][r], r2[j][r], a_log, a_atan);
                slow |= __double2hiint(r2[j][r]) < P2P_SLOW_HI;
              }
            }
            if (__builtin_expect(slow, 0)) {
#pragma unroll
              for (int j = 0; j < NJ; ++j) {
                const int col = c0 + 16 * h + 8 * j + ph;
                const int scol = sym ? sb + col : -1;  // self mode: the column is a target too
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                  const int row = r ? row1 : row0;
                  if (__double2hiint(r2[j][r]) < P2P_SLOW_HI)
                    pr[j][r] = p2p_slow(dx[j][r], dy[j][r], r2[j][r], diag && col == row, tperm, tb + row, scol, st);
                }
              }
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
              a0r = fma(uc[j], pr[j][0].lg, a0r);
              a0i = fma(uc[j], pr[j][0].ag, a0i);
              a1r = fma(uc[j], pr[j][1].lg, a1r);
              a1i = fma(uc[j], pr[j][1].ag, a1i);
              // reversed pairs: same log|z|^2, Arg(-z) = Arg z - pi (Arg z > 0) or + pi (Arg z <= 0)
              const double g0 = pr[j][0].ag, g1 = pr[j][1].ag;
              vr[j] = fma(u0, pr[j][0].lg, u1 * pr[j][1].lg);
              vi[j] = fma(u0, g0 > 0.0 ? g0 - PI : g0 + PI, u1 * (g1 > 0.0 ? g1 - PI : g1 + PI));
            }
          };
          if (two)
            cols(std::integral_constant<int, 2>{});
          else
            cols(std::integral_constant<int, 1>{});
          if (react) {  // the 4 row lanes' partials of the 2 columns, summed below
            s_rs[tl * P2P_RS + ((16 * h + ph) ^ (2 * tl))] = make_double2(vr[0], vi[0]);
            s_rs[tl * P2P_RS + ((16 * h + 8 + ph) ^ (2 * tl))] = make_double2(vr[1], vi[1]);
            hw |= 1u << h;
          }
        }
        if (hw) {  // lane c owns column c of the chunk: add its 4 row-lane partials (fixed order)
          __syncwarp();
          double Rr = 0.0, Ri = 0.0;
          if ((hw >> (lane >> 4)) & 1) {  // pairwise: (r0 + r1) + (r2 + r3)
            double2 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] = s_rs[r * P2P_RS + (lane ^ (2 * r))];
            Rr = (v[0].x + v[1].x) + (v[2].x + v[3].x);
            Ri = (v[0].y + v[1].y) + (v[2].y + v[3].y);
          }
          if (whole) {
            const double2 o = s_re[cb + lane];
            s_re[cb + lane] = make_double2(o.x + Rr, o.y + Ri);
          } else if (write_react && lane < cnt) {
            double2* slot = part + ((int64_t)(sb + c0 + lane) * nslot + qr);
            if (heavy) {
              atomicAdd(&slot->x, Rr);
              atomicAdd(&slot->y, Ri);
            } else if (rc == tk.z) {
              *slot = make_double2(Rr, Ri);
            } else {
              const double2 o = *slot;
              *slot = make_double2(o.x + Rr, o.y + Ri);
            }
          }
        }
        __syncwarp();
      }
      // reduce the 8 phases of each row (lanes tl + 4 ph) through the scratch: lane (tl, ph)
      // stores its two rows' sums; lane L < 16 adds component L & 1 of row L >> 1 over ph
      // (fixed order)
      s_rs[ph * 8 + tl] = make_double2(a0r, a0i);
      s_rs[ph * 8 + 4 + tl] = make_double2(a1r, a1i);
      __syncwarp();
      if (lane < 16) {
        const double* sd_ = (const double*)s_rs;
        const int rr = lane >> 1, comp = lane & 1;
        double a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = sd_[(k * 8 + rr) * 2 + comp];
        const double v = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));  // pairwise
        const int row = rc + (rr & 3) + 4 * (rr >> 2);
        if (row < tk.w) {
          if (sd && whole) {  // rows and reactions of a diagonal block share the slots: add into s_re
            double* re_ = (double*)(s_re + row) + comp;
            *re_ += v;
          } else if (write_rows) {
            double* dst = (double*)(part + (int64_t)(tb + row) * nslot + q) + comp;
            if (sd)  // heavy diagonal: slot shared with the reactions of other row ranges
              atomicAdd(dst, v);
            else
              *dst = v;
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    if (PAIRS && (tk.y & TF_PAIR)) {
      p2p_finish_pair(tk.y, t, tb, tk.w, sb, qr, ns, write_rows, write_react, lo, hi, soff, near, s_re, part, nslot);
    } else if (whole && write_react) {
      if (heavy) {
        for (int i = lane; i < ns; i += 32) {
          double2* slot = part + (int64_t)(sb + i) * nslot + qr;
          atomicAdd(&slot->x, s_re[i].x);
          atomicAdd(&slot->y, s_re[i].y);
        }
      } else {
        for (int i = lane; i < ns; i += 32) part[(int64_t)(sb + i) * nslot + qr] = s_re[i];
      }
    }
    __syncwarp();  // the next task restages s_xy / s_u / s_re
  }
}

// ------------------------------------------------------------------ partial sums + L2P -> Phi
// one warp per target leaf; lanes over its targets; slots added in near-list order
template <int NS>  // slots per target (nslot): all loads of a target issued together
__global__ void __launch_bounds__(128) k_p2p_finish(int64_t lo, int64_t hi, const int32_t* __restrict__ toff,
                                                    const int32_t* __restrict__ nnear, const double2* __restrict__ txy,
                                                    const double2* __restrict__ cen_leaf,
                                                    const double2* __restrict__ loc_leaf, int p,
                                                    const int32_t* __restrict__ tperm,
                                                    const double2* __restrict__ part, int nslot,
                                                    const int32_t* __restrict__ pskip, double2* __restrict__ phi) {
  __shared__ double2 s_loc[4][32];
  const int64_t t = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= hi) return;
  const int tb = toff[t], nt = toff[t + 1] - tb;
  if (nt == 0) return;
  const int nn = nnear[t];
  const unsigned skip = (unsigned)pskip[t];  // slots no task writes (TF_PAIR's q2): read as 0
  const double2 c = cen_leaf[t];
  // the leaf's local expansion in shared memory (one coalesced load), so that the Horner
  // steps below do not wait on a global load each
  double2* const b = s_loc[threadIdx.x >> 5];
  b[lane] = lane <= p ? loc_leaf[t * (p + 1) + lane] : make_double2(0.0, 0.0);
  __syncwarp();
  for (int i = lane; i < nt; i += 32) {
    const int tpos = tb + i;
    double2 v[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q)
      v[q] = (q < nn && !((skip >> q) & 1u)) ? part[(int64_t)tpos * nslot + q] : make_double2(0.0, 0.0);
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int q = 0; q < NS; ++q) {  // near-list order
      re += v[q].x;
      im += v[q].y;
    }
    const double2 y = txy[tpos];
    const double2 z = make_double2(y.x - c.x, y.y - c.y);
    double2 acc = b[p];  // L2P by Horner at y - c_leaf
    for (int k = p - 1; k >= 0; --k) {
      acc = cmul2(acc, z);
      acc.x += b[k].x;
      acc.y += b[k].y;
    }
    phi[tperm[tpos]] = make_double2(acc.x + 0.5 * re, acc.y + im);
  }
}

// ------------------------------------------------------------------ direct sum (NEXT-1)
// Phi_j = sum_i u_i Log(y_j - x_i) over ALL sources (self mode: i != j by index, D16), the
// reference the paper's section-9 error sweeps compare against.  A lane owns one target; the
// block stages 128 sources at a time in shared memory; the same pair math as the near field
// (fast path, exact slow path for |z| < 1e-30).  Coincident pairs (other than i == j in self
// mode) set *bad to the smallest target index involved.
constexpr int DIR_T = 128;
constexpr size_t DIR_SMEM = sizeof(double2) * (P2P_LOG_N + P2P_ATAN_N + DIR_T) + sizeof(double) * DIR_T;
__global__ void __launch_bounds__(DIR_T) k_direct(const double2* __restrict__ sxy, const double* __restrict__ su,
                                                  int64_t n, const double2* __restrict__ txy, int64_t m,
                                                  int self_mode, const double* __restrict__ tabs,
                                                  double2* __restrict__ phi, unsigned long long* bad) {
  extern __shared__ double2 dir_smem[];  // DIR_SMEM bytes: tables, then the staged sources
  double2* s_log = dir_smem;
  double2* s_atan = s_log + P2P_LOG_N;
  double2* s_x = s_atan + P2P_ATAN_N;
  double* s_u = (double*)(s_x + DIR_T);
  p2p_load_tables(tabs, s_log, s_atan);
  const uint32_t a_log = p2p_smem_addr(s_log), a_atan = p2p_smem_addr(s_atan);
  const int64_t j = blockIdx.x * (int64_t)DIR_T + threadIdx.x;
  const bool tv = j < m;
  // canonical +0 imaginary zero of y - x (D13): coordinates read as x + 0
  double2 y = tv ? txy[j] : make_double2(P2P_PAD, P2P_PAD);
  y = make_double2(__dadd_rn(y.x, 0.0), __dadd_rn(y.y, 0.0));
  double re = 0.0, im = 0.0;
  for (int64_t c0 = 0; c0 < n; c0 += DIR_T) {
    __syncthreads();
    const int64_t i = c0 + threadIdx.x;
    if (i < n) {
      const double2 x = sxy[i];
      s_x[threadIdx.x] = make_double2(__dadd_rn(x.x, 0.0), __dadd_rn(x.y, 0.0));
      s_u[threadIdx.x] = su[i];
    } else {
      s_x[threadIdx.x] = make_double2(-P2P_PAD, P2P_PAD);
      s_u[threadIdx.x] = 0.0;
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)DIR_T, n - c0);
    for (int k = 0; k < cnt; ++k) {
      const double2 x = s_x[k];
      const double dx = y.x - x.x, dy = y.y - x.y;
      const double r2 = fma(dx, dx, dy * dy);
      PairOut pr = p2p_fast(dx, dy, r2, a_log, a_atan);
      if (__double2hiint(r2) < P2P_SLOW_HI) {
        if (r2 == 0.0) {
          pr.lg = 0.0;
          pr.ag = 0.0;
          if (tv && !(self_mode && c0 + k == j)) atomicMin(bad, (unsigned long long)j);
        } else {
          pr.lg = 2.0 * log(hypot(dx, dy));
          pr.ag = atan2(__dadd_rn(dy, 0.0), dx);
        }
      }
      re = fma(s_u[k], pr.lg, re);
      im = fma(s_u[k], pr.ag, im);
    }
  }
  if (tv) phi[j] = make_double2(0.5 * re, im);
}

// debug hook: the P2P math on explicit (dx, dy) pairs -> (log |z|^2, Arg z)
__global__ void k_debug_p2p_math(const double2* __restrict__ d, int64_t n, const double* __restrict__ tabs,
                                 double2* __restrict__ out) {
  extern __shared__ double2 dbg_smem[];  // the P2P tables (P2P_TAB_BYTES)
  double2* s_log = dbg_smem;
  double2* s_atan = s_log + P2P_LOG_N;
  p2p_load_tables(tabs, s_log, s_atan);
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dx = d[i].x, dy = __dadd_rn(d[i].y, 0.0);  // canonical +0 imaginary zero (D13)
  const double r2 = fma(dx, dx, dy * dy);
  out[i] = make_double2(p2p_log(r2, p2p_smem_addr(s_log)), p2p_atan2<true>(dy, dx, p2p_smem_addr(s_atan)));
}

}  // namespace

// Pairing of light off-diagonal blocks (TF_PAIR, self mode) pays where leaves average 32-96
// points on a tree of > 2^20 points (column padding and row-step heads halved: C4q -3 %, C4t
// -4 %); elsewhere the pairing
// variant of the kernel only costs (its larger code shifts the register allocation: C4s +2.4 %
// with no pair formed, C5 +1.4 %), so those trees keep the plain kernel.  FMM_P2P_PAIRS=0 / 1
// overrides.
bool fmm_p2p_pairing(const fmm_tree_s* t) {
  if (!t->g.self_mode) return false;
  const char* f = getenv("FMM_P2P_PAIRS");
  if (f && (f[0] == '0' || f[0] == '1')) return f[0] == '1';
  const double mean = (double)t->n / (double)t->g.K;
  return t->n > (1 << 20) && mean >= 32.0 && mean <= 96.0;  // small trees: too few tasks (C2 +16 %)
}

int fmm_build_tasks(fmm_tree_s* t) {
  cudaStream_t s = t->stream;
  const int64_t K = t->g.K;
  const int mode = (t->g.self_mode ? 1 : 0) | (fmm_p2p_pairing(t) ? 2 : 0);
  int32_t* cnt = nullptr;
  size_t sb = fmm_scan_scratch_bytes(K + 1);
  FMM_CUDA_TRY(cudaMallocAsync(&cnt, sizeof(int32_t) * (K + 1) + sb, s));
  k_task_count<<<(unsigned)((K + 1 + 255) / 256), 256, 0, s>>>(K, t->toff, t->soff, t->near, t->nnear, mode,
                                                                t->leaf_lo, t->leaf_hi, cnt);
  int e = fmm_device_scan_i32(cnt, cnt, K + 1, cnt + K + 1, sb, s, &t->launches);
  if (!e)
    k_task_fill<<<(unsigned)((K + 1 + 255) / 256), 256, 0, s>>>(K, t->toff, t->soff, t->near, t->nnear, mode,
                                                                 t->leaf_lo, t->leaf_hi, cnt, t->tasks, t->ntask,
                                                                 t->pskip);
  t->launches += 2;
  cudaFreeAsync(cnt, s);
  FMM_CUDA_TRY(cudaGetLastError());
  return e;
}

int fmm_stage_p2p_pairs(fmm_tree_s* t) {
  const Geo& G = t->g;
  cudaStream_t s = t->stream;
  FMM_CUDA_TRY(cudaMemsetAsync(t->next_task, 0, sizeof(int32_t), s));
  if (G.self_mode) {
    k_heavy_zero<<<148 * 4, 256, 0, s>>>(t->tasks, t->ntask, t->soff, t->near,
                                                                        t->part, G.nslot);
    t->launches++;
  }
  auto launch = [&](auto kern) -> int {
    FMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P2P_SMEM));
    kern<<<148 * P2P_MINB, 32 * P2P_WARPS, P2P_SMEM, s>>>(t->tasks, t->ntask, t->next_task, t->toff, t->soff, t->txy,
                                                           t->sxy, t->su, t->near, t->nnear, t->tperm, t->p2p_tab,
                                                           t->part, fmm_part_slots(G), t->leaf_lo, t->leaf_hi,
                                                           t->status);
    return FMM_OK;
  };
  int e = !G.self_mode ? launch(k_p2p_pairs<false, false>)
                       : (fmm_p2p_pairing(t) ? launch(k_p2p_pairs<true, true>) : launch(k_p2p_pairs<true, false>));
  if (e) return e;
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_stage_p2p_finish(fmm_tree_s* t, double2* phi) {
  const Geo& G = t->g;
  cudaStream_t s = t->stream;
  const int64_t nl = t->leaf_hi - t->leaf_lo;
  if (nl > 0)
    switch (fmm_part_slots(G)) {
#define FMM_FINISH(NS)                                                                                        \
  case NS:                                                                                                    \
    k_p2p_finish<NS><<<(unsigned)((nl * 32 + 127) / 128), 128, 0, s>>>(                                       \
        t->leaf_lo, t->leaf_hi, t->toff, t->nnear, t->txy, t->centre + G.lvl_off[G.L],                        \
        t->loc + G.lvl_off[G.L] * (G.p + 1), G.p, t->tperm, t->part, NS, t->pskip, phi);                        \
    break;
      FMM_FINISH(1)
      FMM_FINISH(7)
      FMM_FINISH(9)
      FMM_FINISH(13)
#undef FMM_FINISH
      default: return FMM_EBADCFG;
    }
  t->launches++;
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_direct_launch(const double* sxy, const double* su, int64_t n, const double* txy, int64_t m, int self_mode,
                      const double* tabs, double* phi, unsigned long long* bad, cudaStream_t s) {
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DIR_SMEM));
  if (m > 0)
    k_direct<<<(unsigned)((m + DIR_T - 1) / DIR_T), DIR_T, DIR_SMEM, s>>>((const double2*)sxy, su, n, (const double2*)txy, m,
                                                                  self_mode, tabs, (double2*)phi, bad);
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}

int fmm_debug_p2p_math_launch(const double* dxdy, int64_t n, const double* tabs, double* out, cudaStream_t s) {
  FMM_CUDA_TRY(cudaFuncSetAttribute(k_debug_p2p_math, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P2P_TAB_BYTES));
  k_debug_p2p_math<<<(unsigned)((n + 255) / 256), 256, P2P_TAB_BYTES, s>>>((const double2*)dxdy, n, tabs, (double2*)out);
  FMM_CUDA_TRY(cudaGetLastError());
  return FMM_OK;
}
