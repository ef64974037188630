// p2p_math.cuh -- FP64 log|z|^2 and Arg z for the P2P near field (kernel Log(y - x)).
//
// Both are table-driven and accurate to ~1 ulp (absolute error below ~2^-52 max(1, |result|));
// they replace libdevice log / atan2, whose integer, branch and polynomial work made the
// pair loop ~4x slower.  Valid for |z| >= 1e-30 (the caller sends
// smaller |z|, including the excluded / coincident z = 0, to an exact slow path).
//
//   log(r2): r2 = 2^k z, z in [0.6875, 1.375); z = c_i (1 + r) with a table of (1/c_i, log c_i)
//            selected by the top mantissa bits: 1024 entries, |r| <= 2^-11 and log1p(r) to r^4
//            (truncation < 2^-57.3 absolute) in the pair kernel; 512 entries, |r| <= 2^-10 and
//            log1p(r) to r^5 (truncation < 2^-62.5) in the M2L's b_0 (a smaller shared-memory copy).
//   atan2  : octant reduction to t = num/den in [0, 1]; t_k = k/64 with k = round(64 t)
//            from a MUFU.RCP64H estimate; atan t = atan t_k + atan q,
//            q = (num - t_k den) / (den + t_k num), |q| <= 1/128 + 2^-20;
//            atan q = q - q^3/3 + q^5/5 - q^7/7 (truncation < 2^-62 |q|);
//            the octant's reference angle and signed slope are tabulated per (oct, k), so
//            that q = (P - tau Q) / (Q + tau P) carries the sign (no fix-up).
//   division: q0 = a r0 from the MUFU.RCP64H estimate r0, q = q0 (1 + e + e^2), e = 1 - b r0,
//            error ~ e^3.
// Polynomial coefficients live in the constant bank (DFMA operands, no register moves).
#pragma once
#include <stdint.h>

#define P2P_LOG_N 1024  // log table of the pair kernel, direct sum and debug hook
#define P2P_LOGC_N 512  // log table of the M2L (compact tables)
#define P2P_TW 8  // targets per P2P warp task
#define P2P_G 4   // source phases per task (P2P_TW * P2P_G = 32 lanes)
#define P2P_ATAN_K 64    // M2L (compact table): t_k = k / 64, k = 0..64
#define P2P_ATAN_KS 256  // pair kernel (sparse table): t_k = k / 256, k = 0..255 (256 clamps to 255)
// table layout (doubles): [0, 2N) log (1/c, log c) pairs; then (theta[oct][k], tau[oct][k])
#define P2P_ATAN_SUB 256  // entries per octant sub-table of the sparse layout
#define P2P_ATAN_N (8 * P2P_ATAN_SUB)
#define P2P_TAB_LOG 0
#define P2P_TAB_ATAN (2 * P2P_LOG_N)
#define P2P_TAB_ATANC (2 * P2P_LOG_N + 2 * P2P_ATAN_N)  // compact copy: entry oct * 65 + k
#define P2P_TAB_LOGC (P2P_TAB_ATANC + 2 * 8 * (P2P_ATAN_K + 1))  // the 512-entry log table
#define P2P_TAB_DOUBLES (P2P_TAB_LOGC + 2 * P2P_LOGC_N)

// atan table entry of (octant, k), octant bit 0 = swap, bit 1 = dx < 0, bit 2 = dy < 0:
// k + 256 [dx < 0] + 512 [dy < 0] + 1024 [swap], so that the pair kernel forms the index from
// the sign bytes of dx, dy with one PRMT (p2p_atan2<true>)
__host__ __device__ inline int p2p_atan_index(int oct, int k) {
  return k + P2P_ATAN_SUB * ((oct >> 1) & 1) + 2 * P2P_ATAN_SUB * ((oct >> 2) & 1) + 4 * P2P_ATAN_SUB * (oct & 1);
}
// |z|^2 below this (hi word of 1e-60) takes the exact slow path
#define P2P_SLOW_HI 0x3379b604
// z intervals of an N-entry table: bit patterns [OFF + i 2^S, OFF + (i+1) 2^S), S = 52 - log2 N,
// OFF = 0x3fe6000000000000 - 2^(S-1), so that the bit pattern of 1.0 is the centre of interval
// 0.625 N (one binade of bit patterns covers z in [0.6875, 1.375))
template <int N>
struct P2PLogTab;
template <>
struct P2PLogTab<1024> {
  static constexpr int SHIFT = 42, OFF_HI = 0x3fe5fe00;
  static constexpr unsigned long long OFF = 0x3fe5fe0000000000ull;
};
template <>
struct P2PLogTab<512> {
  static constexpr int SHIFT = 43, OFF_HI = 0x3fe5fc00;
  static constexpr unsigned long long OFF = 0x3fe5fc0000000000ull;
};

__constant__ double P2P_C[13] = {
    1.0 / 7.0, -1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -0.5,  // log1p Taylor r^7 .. r^2
    1.0 / 9.0, -1.0 / 7.0, 1.0 / 5.0, -1.0 / 3.0,                   // atan Taylor q^9 .. q^3
    0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45,                     // ln 2 = hi (42 bits) + lo
    0x1.62e42fefa39efp-1                                             // ln 2 (double)
};

// copy the tables to shared memory (whole block; ends with __syncthreads)
// s_log[P2P_LOG_N], s_atan[P2P_ATAN_N] (the layout of p2p_atan_index)
__device__ __forceinline__ void p2p_load_tables(const double* __restrict__ tabs, double2* s_log, double2* s_atan) {
  const double2* t2 = (const double2*)tabs;
  for (int i = threadIdx.x; i < P2P_LOG_N; i += blockDim.x) s_log[i] = t2[P2P_TAB_LOG / 2 + i];
  for (int i = threadIdx.x; i < P2P_ATAN_N; i += blockDim.x) s_atan[i] = t2[P2P_TAB_ATAN / 2 + i];
  __syncthreads();
}

__device__ __forceinline__ double p2p_rcp(double b) {
  double r0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(b));
  double e = fma(-b, r0, 1.0);
  e = fma(e, e, e);
  return fma(e, r0, r0);
}

// 16-byte load from a 32-bit shared-space address
__device__ __forceinline__ double2 p2p_lds2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// entry i of a table of double2: a 32-bit shared-space address (the pair kernel, direct sum and
// debug hook keep their tables in shared memory) or a global pointer (the M2L's few Log terms per
// cell read the tables through L1 instead of staging 16 KB of them per block)
__device__ __forceinline__ double2 p2p_tab_entry(uint32_t smem_addr, uint32_t i) { return p2p_lds2(smem_addr + 16 * i); }
__device__ __forceinline__ double2 p2p_tab_entry(const double2* __restrict__ gtab, uint32_t i) { return __ldg(gtab + i); }

// shared-space address of a table, laundered through an opaque move so that the compiler keeps
// it in a register instead of re-deriving the shared window address at every use
__device__ __forceinline__ uint32_t p2p_smem_addr(const void* p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}

// log(r2) = kd * ln 2 + lz for a normal r2 >= 1e-60 (N-entry log table in shared memory).
// The N intervals of z are centred so that z = 1 is the centre of its interval
// (c = 1, 1/c = 1, log c = 0): log(1) = 0 exactly, which the self-pair exclusion relies on.
template <int N = P2P_LOG_N, class TAB = uint32_t>
__device__ __forceinline__ void p2p_log_split(double r2, TAB logtab, double* kd, double* lz) {
  using T = P2PLogTab<N>;
  int hi = __double2hiint(r2), lo = __double2loint(r2);
  int tmp = hi - T::OFF_HI;
  int i = (tmp >> (T::SHIFT - 32)) & (N - 1);
  int k = tmp >> 20;  // arithmetic shift
  double z = __hiloint2double(hi - (tmp & 0xfff00000), lo);
  const double2 cl = p2p_tab_entry(logtab, (uint32_t)i);  // (1/c_i, log c_i)
  double r = fma(z, cl.x, -1.0);
  double r_2 = r * r;
  double q;
  if (N >= 1024) {
    // |r| <= 2^-11: log1p(r) = r - r^2/2 + r^3/3 - r^4/4, truncation r^5/5 < 2^-57.3
    q = fma(r, -0.25, P2P_C[4]);  // 1/3 (full precision)
  } else {
    // r^5 coefficient rounded to a 20-bit mantissa (SASS immediate): its error
    // (< 2^-21 relative) times r^5/5 stays below 2^-70 for |r| <= 2^-10
    q = fma(r, 0x1.9999900000000p-3 /* ~1/5 */, -0.25);
    q = fma(q, r, P2P_C[4]);  // 1/3 (full precision)
  }
  q = fma(q, r, -0.5);
  *lz = cl.y + fma(r_2, q, r);  // log c_i + log1p(r)
  *kd = (double)k;
}

template <int N = P2P_LOG_N, class TAB = uint32_t>
__device__ __forceinline__ double p2p_log(double r2, TAB logtab) {
  double kd, lz;
  p2p_log_split<N, TAB>(r2, logtab, &kd, &lz);
  return fma(kd, P2P_C[10], lz) + kd * P2P_C[11];
}

// Arg(dx + i dy) in (-pi, pi] for |z| >= 1e-30.  dy must not be -0: callers pass a
// canonical +0 imaginary zero (D13; the sorted coordinates are canonicalised at the gather,
// so y - x never yields -0 there).
// SPARSE: atab holds P2P_ATAN_N entries in the p2p_atan_index layout with knots k / 256 (pair
// kernel, direct sum, debug hook): |q| <= 1/512, atan q to q^5 (truncation < 2^-56.8 |q|);
// else the compact 8 x 65 copy with knots k / 64 (M2L), where k must be <= 64 (|z| normal):
// |q| <= 1/128, atan q to q^7
template <bool SPARSE, class TAB = uint32_t>
__device__ __forceinline__ double p2p_atan2(double dy, double dx, TAB atab) {
  // Rotation by the reference direction theta of (octant, k): with (P, Q) = (dy, dx), or
  // (-dx, dy) when |dy| > |dx|, and the table's signed slope tau (+-k/64; its sign folds the
  // octant's orientation), Arg z = theta + atan(q), q = (P - tau Q) / (Q + tau P) -- no sign
  // fix-up.  k = round(K |P| / |Q|) from the MUFU reciprocal (~2^-22) and the 1.5 2^52 shift.
  // swap = |dy| > |dx|, decided in FP32 on the high words (sign, 11-bit exponent, 20 mantissa
  // bits read as a float: monotonic in the magnitude for |x| < 2^1017) instead of a DSETP on the
  // FP64 pipe; a tie in the high words leaves swap false with |P| / |Q| < 1 + 2^-20, which the
  // sparse table's k <= 255 clamp covers (|q| <= 1/512 + 2^-20).  The compact (M2L) path keeps
  // the exact test (its k is masked, not clamped).
  const int hx0 = __double2hiint(dx), hy0 = __double2hiint(dy);
  const bool swap = SPARSE ? fabsf(__int_as_float(hy0)) > fabsf(__int_as_float(hx0)) : fabs(dy) > fabs(dx);
  // -dx by a sign-bit flip of the high word (an ALU op, not a DADD on the FP64 pipe)
  const double ndx = __hiloint2double(hx0 ^ (int)0x80000000, __double2loint(dx));
  const double P = swap ? ndx : dy, Q = swap ? dy : dx;
  double r0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(Q));
  const int k = __double2loint(fma(fabs(P * r0), SPARSE ? (double)P2P_ATAN_KS : (double)P2P_ATAN_K,
                                   6755399441055744.0));  // 0..K (clamped / masked below)
  const int hx = __double2hiint(dx), hy = __double2hiint(dy);
  uint32_t idx;
  if (SPARSE) {
    // byte 0 = sign of dx replicated (bit 7), byte 1 = sign of dy (bit 8), shifted to +256 / +512;
    // k = 256 (t = 1 within rounding) and the garbage k of |z| < 1e-30 clamp to 255 (|q| <= 1/512)
    uint32_t sg;
    asm("prmt.b32 %0, %1, %2, 0xFB;" : "=r"(sg) : "r"(hx), "r"(hy));
    idx = ((sg & 0x180u) << 1) + min((uint32_t)k, (uint32_t)(P2P_ATAN_SUB - 1)) + (swap ? 4u * P2P_ATAN_SUB : 0u);
  } else {
    // octant: bit0 swap, bit1 dx < 0, bit2 dy < 0
    const int oct = (int)swap | (((unsigned)hx >> 30) & 2) | (((unsigned)hy >> 29) & 4);
    idx = oct * (P2P_ATAN_K + 1) + (k & 0x7f);
  }
  const double2 Tt = p2p_tab_entry(atab, idx);  // (theta[oct][k], tau[oct][k])
  const double a = fma(-Tt.y, Q, P);
  const double b = fma(Tt.y, P, Q);
  // q = a / b: q0 = a r0 beside the residual e = 1 - b r0, then q0 (1 + e + e^2)
  double r1;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r1) : "d"(b));
  const double q0 = a * r1;
  double e = fma(-b, r1, 1.0);
  e = fma(e, e, e);
  const double q = fma(q0, e, q0);
  const double q2 = q * q;
  double Pq;
  if (SPARSE) {
    Pq = fma(q2, P2P_C[8] /* 1/5 */, P2P_C[9] /* -1/3 */);
  } else {
    // q^7 coefficient rounded to a 20-bit mantissa (immediate), error < 2^-62 |q|
    Pq = fma(q2, -0x1.2492400000000p-3 /* ~-1/7 */, P2P_C[8] /* 1/5 */);
    Pq = fma(Pq, q2, P2P_C[9]);  // -1/3
  }
  return Tt.x + fma(q * q2, Pq, q);
}
