// thmm_kernels.cuh -- sm_100a kernels of the HMM forward log-likelihood.
//
// The likelihood is the ordered product (reference core.py:7, engine.py:3-11)
//     L = delta' (Gamma P(x_0)) (Gamma P(x_1)) ... (Gamma P(x_{N-1})) 1.
// The chain is cut into contiguous segments (reference segment_bounds,
// engine.py:97-111).  Each segment is reduced to a K x K scaled product with
// FP64 tensor-core MMAs (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4; tcgen05 has
// no f64 kind), with the emission diagonal evaluated in-kernel from the raw
// (present, lon, lat) stream and never written to HBM.  Segment products are
// then folded by a log-depth tree of the same MMA machinery and finished
// against delta.
//
// Register-resident chaining.  For one 8-row tile of the running product M,
// an m8n8k4 accumulator fragment holds, in lane (g = lane/4, q = lane%4),
// the two entries M[g][8n + 2q + h], h = 0, 1.  The A fragment of the next
// step needs, in the same lane, A[g][k = q].  Choosing the k-order of the
// contraction so that k-chunk (nb, h) covers the states 8nb + 2q + h makes
// A-chunk (nb, h) exactly the lane's own accumulator entry (nb, h): the
// product never leaves registers and no shuffles are needed.  The B operand
// (Gamma, fixed for the whole chain) is stored in shared memory in that
// permuted fragment order, one 16-byte (h=0, h=1) pair per lane, so each
// (n-tile, k-pair) costs one conflict-free LDS.128 for two MMAs.
//
// Row stacking.  The rows of a segment product are independent forward
// recursions that share Gamma (rows of M = e_r' Gamma P(x_lo) ...).  A CTA
// therefore stacks the K rows of G consecutive segments into one tall
// G*K-row operand, padded only once to the warp tile (8 rows) and to a warp
// count that is a multiple of 4 so the four SM sub-partitions (one DMMA unit
// each) carry equal work.  Each lane reads the emission row of its own
// segment in the epilogue.
//
// Scaling.  Instead of dividing by the running max and adding log(max)
// (reference engine.py:145-150), rows are rescaled by exact powers of two
// (ilogb of the row max) and the exponents are summed exactly; renormalising
// therefore introduces no rounding at all, and each row carries its own
// exponent so one small row cannot underflow because another row is large.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace thmm {

constexpr int kEmissionBlock = 32;   // steps of emissions staged in smem at a time (small K)
// Steps per emission block of the FP64 chain kernel: 64 for wide rows (one
// CTA per SM, shared memory to spare; half the block barriers and record
// stagings), 32 where two CTAs per SM must fit.
__host__ __device__ constexpr int chain_eb(int nt) { return nt >= 6 ? 2 * kEmissionBlock : kEmissionBlock; }
constexpr unsigned kFull = 0xffffffffu;

// Threads per chain CTA allowed by __launch_bounds__ (caps registers per thread
// at 65536 / threads): wide CTAs only where the fragments are small.
__host__ __device__ constexpr int chain_max_threads(int nt) {
  return nt <= 4 ? 512 : (nt <= 6 ? 768 : 640);
}

// "Lean" chain variants (padded K <= 32): the B fragments and tail couplings
// are re-read from shared memory every step instead of being hoisted into
// registers, which keeps a thread at <= 64 registers so two 16-warp CTAs fit
// per SM -- the DMMA/FP64 pipe needs that many warps to stay busy when each
// warp's step is only a few dozen MMAs long.
__host__ __device__ constexpr bool chain_lean(int nt) { return nt <= 4; }
__host__ __device__ constexpr int chain_min_blocks(int nt) { return chain_lean(nt) ? 2 : 1; }

struct StateParams {
  const double* gamma;   // [B][K][K]
  const double* states;  // [8][B][K]: p, q, mu0, mu1, l00, l10, l11, log_det
  const double* delta;   // [B][K]
};

struct ChainArgs {
  const uint8_t* present;
  const double* lon;
  const double* lat;
  int64_t lo;        // first record of the range
  int64_t n;         // records in the range
  int64_t nseg;      // segments per proposal
  int K;
  int B;
  int G;             // segments stacked per CTA
  int period;        // renormalisation period (>= 1)
  double neg_log_2pi;
  StateParams P;
  double* seg_m;     // [B][nseg][KP][KP]
  double* seg_e;     // [B][nseg]  base-2 exponent of each node
  int64_t node_stride_b;  // nodes per proposal in seg_m/seg_e (>= nseg; several ranges may share them)
  int64_t node_offset;    // index of this range's first segment node
  int x3;                 // TF32 tensor-core chain only: operand split (0 tf32, 1 3xTF32, 2 2xTF32)
  long long* trace;       // debug only (tools/tc_trace.cu): per-step clock64 stamps; nullptr otherwise
  int sysmem;             // records live in pinned host memory (zero-copy): uncached PCIe loads
  // Rank-one collapse (thmm_vec.cuh), run-absorbing chain only: > 0 enables
  // the per-window test; the collapse state is indexed like the nodes.
  double collapse_tol;
  double* col_r;          // [node][KPE] pivot row, normalised to max in [1, 2)
  double* col_d;          // [node][KPE] row exponent offsets e_i - e_p (<= 0; -inf: zero row)
  double* col_c;          // [node][KPE] row ratios rho_i (row i = rho_i 2^d_i r)
  double* col_meta;       // [node][2] records consumed at the collapse (-1: full node written), pivot exponent
  int collapse_win;       // records between rank-one tests (1..32)
  // Stitched chain (thmm_vec.cuh): per node the final normalised row of the
  // main pass and its exponent, the link term of segment s >= 1, and a
  // per-proposal flag set when a link did not converge.
  double* fin;            // [node][KPE]
  double* fin_e;          // [node]
  double* link;           // [node]
  int* link_fail;         // [B]
  int stitch_delta;       // segment 0 starts from delta (the range is the whole chain)
  const double* link_src; // link kernel, external mode: segment 0 only, p from these rows (another rank's final row)
  int64_t link_src_stride;
  double* link_out;       // external mode: [B][2] link term, fail flag
  // Stitched main pass split in time (records staged by DMA while the chain
  // runs): launch t_chunk of t_chunks covers records [time_chunk_begin(L, c),
  // time_chunk_begin(L, c+1)) of every segment (L its length) and carries the
  // rows in fin / fin_e.
  int t_chunk;
  int t_chunks;           // <= 1: one launch over the whole segment
  double t_frac[17];      // chunk c starts at record floor(L t_frac[c]) of its segment (t_frac[t_chunks] = 1)
  // Single-launch staged main pass: the copy stream bumps *arrive to c + 1
  // once time chunk c has landed (stream memory operation); the kernel covers
  // whole segments and waits per record window for the chunk it needs.
  const unsigned* arrive;
  // Row-stacked kernels: Gamma already in the B-fragment entry layout,
  // [B][runs_entry_pairs] (entry_prep_kernel), copied into shared memory with
  // one bulk (TMA) copy per CTA; nullptr: each CTA permutes Gamma itself.
  const double2* gent;
  // Row-stacked kernels: 1 = emissions of the events of 8 steps at a time
  // (batched, 4 independent chains per lane) into a per-warp buffer of 64
  // rows -- launches spread thin over the SMs, where a lone warp is latency-
  // bound; 0 = per step (full waves, FP64-pipe-bound).
  int ebatch;
};

struct FoldArgs {
  const double* in_m;   // node (b, i) at in_m + (i*stride_i + b*stride_b) * KP*KP
  const double* in_e;   //          and in_e[i*stride_i + b*stride_b]
  int64_t stride_i;
  int64_t stride_b;
  int64_t n_in;         // nodes per proposal
  int64_t n_out;        // groups per proposal (segment_bounds(n_in, n_out))
  double* out_m;        // [B][n_out][KP][KP]
  double* out_e;        // [B][n_out]
  int K;
  int B;
  int finish;           // n_out == 1: also evaluate log(delta' m 1) + e ln 2
  const double* delta;  // [B][K]
  double* loglik;       // [B]
  int32_t* status;      // [B]
};

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// One 16-byte B-fragment pair from shared memory, re-read every step: Gamma
// stays in shared memory instead of pinning 4*NT^2 registers, which keeps the
// register budget small enough for wide (many-warp) CTAs.
__device__ __forceinline__ double2 lds_f64x2(const double2* p) {
  double2 v;
  const unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(p));
  // ld.volatile: ptxas must not hoist the loop-invariant load out of the step loop
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// 2^n for n in [-1022, 1023], exact.
__device__ __forceinline__ double pow2_normal(int n) {
  return __longlong_as_double(static_cast<long long>(n + 1023) << 52);
}

// x * 2^n exactly (or correctly underflowed) for n in [-2044, 2046].
__device__ __forceinline__ double scale_pow2(double x, int n) {
  if (n > 1023) return (x * pow2_normal(1023)) * pow2_normal(n - 1023);
  if (n < -1022) return (x * pow2_normal(-1022)) * pow2_normal(n < -2044 ? -1022 : n + 1022);
  return x * pow2_normal(n);
}

// Segment bounds of reference engine.py:97-111: earlier blocks take the remainder.
__device__ __forceinline__ void segment_range(int64_t n, int64_t nseg, int64_t s, int64_t& lo,
                                              int64_t& hi) {
  const int64_t base = n / nseg, rem = n % nseg;
  lo = s * base + (s < rem ? s : rem);
  hi = lo + base + (s < rem ? 1 : 0);
}

// acc[nt][h] = sum_k A[k-chunk] * B[chunk][nt]  (one 8-row tile, all NT n-tiles).
// SKIP: the last k-chunk (nb = NT-1, h = 1) holds only padding states (K % 8 == 1).
template <int NT, bool SKIP, bool LEAN = false>
__device__ __forceinline__ void tile_product(double (&acc)[NT][2], const double (&a)[NT][2],
                                             const double2* __restrict__ bsm, int lane) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  // n-tiles in groups of up to 4: consecutive MMAs target different
  // accumulators, so a dependent MMA is >= 3 issues behind its predecessor
  // (DMMA latency ~26 cycles vs 16 cycles per issue per sub-partition).
  constexpr int GRP = NT < 4 ? NT : 4;
#pragma unroll
  for (int nb = 0; nb < NT; ++nb) {
    const bool h1 = !(SKIP && nb == NT - 1);
#pragma unroll
    for (int n0 = 0; n0 < NT; n0 += GRP) {
      double2 bf[GRP];
#pragma unroll
      for (int j = 0; j < GRP; ++j)
        if (n0 + j < NT)
          bf[j] = LEAN ? lds_f64x2(bsm + ((n0 + j) * NT + nb) * 32 + lane) : bsm[((n0 + j) * NT + nb) * 32 + lane];
#pragma unroll
      for (int j = 0; j < GRP; ++j)
        if (n0 + j < NT) dmma_m8n8k4(acc[n0 + j][0], acc[n0 + j][1], a[nb][0], bf[j].x);
      if (h1) {
#pragma unroll
        for (int j = 0; j < GRP; ++j)
          if (n0 + j < NT) dmma_m8n8k4(acc[n0 + j][0], acc[n0 + j][1], a[nb][1], bf[j].y);
      }
    }
  }
}

// lds_f64x2 at a shared-memory address already in the shared window (the
// row-stacked kernels compute their entry's address once, not per step).
__device__ __forceinline__ double2 lds_f64x2_at(unsigned addr) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// tile_product with the B fragments addressed from `base_lane` = shared
// address of the entry + 16 * lane.
template <int NT, bool SKIP>
__device__ __forceinline__ void tile_product_at(double (&acc)[NT][2], const double (&a)[NT][2], unsigned base_lane) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  constexpr int GRP = NT < 4 ? NT : 4;
#pragma unroll
  for (int nb = 0; nb < NT; ++nb) {
    const bool h1 = !(SKIP && nb == NT - 1);
#pragma unroll
    for (int n0 = 0; n0 < NT; n0 += GRP) {
      double2 bf[GRP];
#pragma unroll
      for (int j = 0; j < GRP; ++j)
        if (n0 + j < NT) bf[j] = lds_f64x2_at(base_lane + static_cast<unsigned>(((n0 + j) * NT + nb) * 32 * 16));
#pragma unroll
      for (int j = 0; j < GRP; ++j)
        if (n0 + j < NT) dmma_m8n8k4(acc[n0 + j][0], acc[n0 + j][1], a[nb][0], bf[j].x);
      if (h1) {
#pragma unroll
        for (int j = 0; j < GRP; ++j)
          if (n0 + j < NT) dmma_m8n8k4(acc[n0 + j][0], acc[n0 + j][1], a[nb][1], bf[j].y);
      }
    }
  }
}

// Max over the row held by the 4 lanes of a quad.
template <int NT>
__device__ __forceinline__ double row_max(const double (&a)[NT][2]) {
  double mx = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(a[nt][0], a[nt][1]));
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 2));
  return mx;
}

// Multiply a row by 2^-ex exactly.
template <int NT>
__device__ __forceinline__ void scale_row(double (&a)[NT][2], int ex) {
  if (ex >= -1022 && ex <= 1022) {
    const double s = pow2_normal(-ex);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      a[nt][0] *= s;
      a[nt][1] *= s;
    }
  } else {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      a[nt][0] = scale_pow2(a[nt][0], -ex);
      a[nt][1] = scale_pow2(a[nt][1], -ex);
    }
  }
}

// Rescale a row so its max lies in [1, 2); adds the exponent to rexp.
template <int NT>
__device__ __forceinline__ void renorm_row(double (&a)[NT][2], double& rexp) {
  const double mx = row_max<NT>(a);
  if (mx > 0.0) {
    const int ex = ilogb(mx);
    scale_row<NT>(a, ex);
    rexp += static_cast<double>(ex);
  }
}

// Block-wide reductions (all threads get the result; fixed order).
__device__ __forceinline__ double block_max(double v, double* red, int nwarps) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < nwarps; ++w) r = fmax(r, red[w]);
  return r;
}

__device__ __forceinline__ double block_sum(double v, double* red, int nwarps) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < nwarps; ++w) r += red[w];
  return r;
}

// Stage a K x K row-major matrix (leading dim ld) as permuted B fragments.
template <int NT>
__device__ __forceinline__ void stage_b_fragments(double2* bsm, const double* __restrict__ m, int K,
                                                  int ld) {
  for (int idx = threadIdx.x; idx < NT * NT * 32; idx += blockDim.x) {
    const int l = idx & 31, pair = idx >> 5;
    const int nb = pair % NT, nt = pair / NT;
    const int k0 = 8 * nb + 2 * (l & 3), col = 8 * nt + (l >> 2);
    double v0 = 0.0, v1 = 0.0;
    if (col < K) {
      if (k0 < K) v0 = m[k0 * ld + col];
      if (k0 + 1 < K) v1 = m[(k0 + 1) * ld + col];
    }
    bsm[idx] = make_double2(v0, v1);
  }
}

// The 8 per-state emission constants of one state, held in registers, plus
// the correctly rounded reciprocals of the two Cholesky divisors.
struct StateConsts {
  double p, q, mu0, mu1, l00, l10, l11, c, r00, r11;
};

__device__ __forceinline__ StateConsts load_state_consts(const double* pj, int kp) {
  const double l00 = pj[4 * kp], l11 = pj[6 * kp];
  return StateConsts{pj[0], pj[kp], pj[2 * kp], pj[3 * kp], l00, pj[5 * kp], l11, pj[7 * kp],
                     __drcp_rn(l00), __drcp_rn(l11)};
}

// a / b from the correctly rounded reciprocal r of b: one Newton correction of
// a*r (Markstein), which returns the correctly rounded quotient for all but
// rare boundary cases (then within one ulp) -- 3 FP64 ops instead of the
// ~10-op IEEE division sequence, in the chain kernels' emission stage.
__device__ __forceinline__ double div_via_rcp(double a, double b, double r) {
  const double q = __dmul_rn(a, r);
  const double e = __fma_rn(-q, b, a);
  return __fma_rn(e, r, q);
}

// 2^(j/64), j = 0..63, correctly rounded (computed at 60 digits).
__device__ const double kExp2Tab64[64] = {0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0, 0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0, 0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0, 0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0, 0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0, 0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0, 0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0, 0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0, 0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0, 0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0, 0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0, 0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0, 0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0, 0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0, 0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0, 0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};

// e^x, table-driven and branch-free: x = (64 m + j) ln2/64 + r with
// |r| <= ln2/128 (two-part ln2/64, the high part exact for |k| < 2^17),
// e^r by its Taylor series to r^5 (truncation < 4e-17 relative), times
// 2^(j/64) from the table and 2^m as two exact power-of-two factors (gradual
// underflow below 2^-1022); x clamped to [-746, 709.7].  ~10 FP64 operations
// and no branch, so the emissions of several rows interleave.
// `tab`: kExp2Tab64 or a shared-memory copy of it.  The clamp is a plain
// select (the argument is never NaN).
//
// FP64-pipe economy (the DMMAs share that pipe): the range clamp is taken
// only when the high word says |x| >= ~709.6 (an integer compare; the same
// clamped value as a two-sided select), the integer k comes from the low word
// of fma(x, 64/ln2, 1.5 * 2^52) (round-to-nearest of the exact product; no
// F2I), and 2^m is applied by adding m to the exponent field whenever the
// result is normal (the two-multiply scaling only for results below
// 2^-1020).  Values: as the two-multiply form, except k may differ by one when
// x 64/ln2 lies within an ulp of a half-integer (still |r| <= ln2/128 + ulp).
__device__ __forceinline__ double exp_tab(double x, const double* tab = kExp2Tab64) {
  double xc = x;
  if ((__double2hiint(x) & 0x7fffffff) >= 0x40862D00) xc = x < -746.0 ? -746.0 : (x > 709.7 ? 709.7 : x);
  const double kdm = fma(xc, 92.33248261689366, 0x1.8p52);  // x 64 / ln 2 + 1.5 * 2^52
  const double kd = kdm - 0x1.8p52;
  const int k = __double2loint(kdm);
  double r = fma(kd, -0x1.62e42fefa0000p-7, xc);
  r = fma(kd, -2.572804622327669e-14, r);
  double p = fma(r, 8.3333333333333332e-03, 4.1666666666666664e-02);
  p = fma(p, r, 0.16666666666666666);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int m = k >> 6;
  const double tp = tab[k & 63] * p;
  if (m >= -1020) return __hiloint2double(__double2hiint(tp) + (m << 20), __double2loint(tp));
  const int m1 = max(m, -1000);
  return (tp * pow2_normal(m1)) * pow2_normal(m - m1);
}

// Emission diagonal entry from register constants (the arithmetic of
// emission(), divisions refined from reciprocals, exp_tab).
__device__ __forceinline__ double emission_rc(bool present, double x, double y, const StateConsts& k,
                                              const double* tab = kExp2Tab64) {
  if (!present) return k.q;
  const double z0 = div_via_rcp(__dsub_rn(x, k.mu0), k.l00, k.r00);
  const double z1 = div_via_rcp(__dsub_rn(__dsub_rn(y, k.mu1), __dmul_rn(k.l10, z0)), k.l11, k.r11);
  const double quad = __dadd_rn(__dmul_rn(z0, z0), __dmul_rn(z1, z1));
  return __dmul_rn(k.p, exp_tab(__dsub_rn(k.c, __dmul_rn(0.5, quad)), tab));
}

// Emission diagonal entry (reference core.py:255-258, same operation order).
// pj points at the 8 per-state constants of state j with stride kp:
// p, q, mu0, mu1, l00, l10, l11, c = -log(2 pi) - 0.5 log_det.
__device__ __forceinline__ double emission(bool present, double x, double y, const double* pj, int kp) {
  if (!present) return pj[kp];
  const double z0 = __ddiv_rn(__dsub_rn(x, pj[2 * kp]), pj[4 * kp]);
  const double z1 = __ddiv_rn(__dsub_rn(__dsub_rn(y, pj[3 * kp]), __dmul_rn(pj[5 * kp], z0)), pj[6 * kp]);
  const double quad = __dadd_rn(__dmul_rn(z0, z0), __dmul_rn(z1, z1));
  return __dmul_rn(pj[0], exp(__dsub_rn(pj[7 * kp], __dmul_rn(0.5, quad))));
}

// Records of one emission block, staged in shared memory: x[G*EB], y[G*EB]
// (f64) and flag[G*EB] (0 quiet, 1 event, 2 no record).
struct RecordStage {
  double* x;
  double* y;
  uint8_t* flag;
};

__host__ __device__ constexpr size_t record_stage_bytes(int G, int EB) {
  return static_cast<size_t>(G) * EB * 17 + 16;
}

// Shared-memory footprint of the chain kernel: NT DMMA head tiles plus TAIL
// SIMT tail states (0 = none), G stacked segments, `warps` warps.
__host__ __device__ constexpr size_t chain_smem_bytes(int nt, int tail, int G, int warps) {
  return static_cast<size_t>(nt) * nt * 32 * 16 +                                  // B fragments
         static_cast<size_t>(2) * tail * nt * 4 * 16 +                             // tail coupling pairs
         static_cast<size_t>(2) * G * chain_eb(nt + (tail > 0)) * 8 * (nt + (tail > 0)) * 8 + // emission blocks (x2)
         static_cast<size_t>(8) * 8 * (nt + (tail > 0)) * 8 +                      // emission constants
         static_cast<size_t>(tail) * tail * 8 +                                    // tail-tail block
         static_cast<size_t>(8) * warps * 8 +                                      // row exponents
         static_cast<size_t>(16) * G +                                             // segment table
         record_stage_bytes(G, chain_eb(nt + (tail > 0)));                         // staged records
}

// Carve a RecordStage at `p` (rounded up to 8 bytes).
__device__ __forceinline__ RecordStage record_stage_at(void* p, int G, int EB) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 7) & ~static_cast<uintptr_t>(7);
  double* x = reinterpret_cast<double*>(a);
  return RecordStage{x, x + G * EB, reinterpret_cast<uint8_t*>(x + 2 * G * EB)};
}

// Record t of the stream: returns present; lon/lat are read for present
// records only (an absent record's coordinates are placeholders, never used).
// sysmem: the stream is pinned host memory read in place over PCIe
// (zero-copy); ld.global.cv fetches it afresh on every call rather than
// trusting a cached line.
__device__ __forceinline__ bool load_record(const ChainArgs& a, int64_t t, double& x, double& y) {
  bool p;
  if (a.sysmem) {
    p = __ldcv(a.present + t) != 0;
    x = p ? __ldcv(a.lon + t) : 0.0;
    y = p ? __ldcv(a.lat + t) : 0.0;
  } else {
    p = a.present[t] != 0;
    x = p ? a.lon[t] : 0.0;
    y = p ? a.lat[t] : 0.0;
  }
  return p;
}

// The present flag of record t (as load_record).
__device__ __forceinline__ bool load_flag(const ChainArgs& a, int64_t t) {
  return (a.sysmem ? __ldcv(a.present + t) : a.present[t]) != 0;
}

// Stage records [t0, t0 + cnt) of the CTA's segments: one thread per
// (segment, step) issues the three global loads, so the block pays ONE
// global-memory latency instead of one per emission a thread evaluates.
// END_ALIGNED: segment s consumes record start + t - (len_max - len_s)
// (tensor-core kernel), else record start + t.  Ends with a CTA barrier.
template <int EB, bool END_ALIGNED>
__device__ __forceinline__ void stage_records(const ChainArgs& args, const RecordStage& rs, const int64_t* sseg,
                                              int64_t t0, int cnt, int g_eff, int64_t len_max) {
  for (int idx = threadIdx.x; idx < g_eff * EB; idx += blockDim.x) {
    const int s = idx / EB, i = idx - s * EB;
    const int64_t len = sseg[2 * s + 1];
    const int64_t ts = END_ALIGNED ? t0 + i - (len_max - len) : t0 + i;
    const bool ok = i < cnt && ts >= 0 && ts < len;
    uint8_t f = 2;
    double x = 0.0, y = 0.0;
    if (ok) f = load_record(args, sseg[2 * s] + ts, x, y) ? 1 : 0;
    rs.flag[idx] = f;
    rs.x[idx] = x;
    rs.y[idx] = y;
  }
  __syncthreads();
}

// Emission block [t0, t0 + EB) of the CTA's G stacked segments into buf[s][i][j]
// (zero for padding states and for steps past a segment's end).
template <int KP, int EB>
__device__ __noinline__ void fill_emission_block(const ChainArgs& args, double* buf, const double* psm,
                                                    const int64_t* sseg, int64_t t0, int64_t len_max,
                                                    int g_eff, RecordStage rs) {
  const int cnt = static_cast<int>(len_max - t0 < EB ? len_max - t0 : EB);
  stage_records<EB, false>(args, rs, sseg, t0, cnt, g_eff, len_max);
  // Thread -> one state j (constants in registers), records strided by
  // blockDim / KP; compile-time divisors only.
  const int j = threadIdx.x % KP;
  const int rstride = blockDim.x / KP;
  if (static_cast<int>(threadIdx.x) >= rstride * KP) return;
  const bool real = j < args.K;
  const StateConsts kc = load_state_consts(psm + j, KP);
  for (int r = threadIdx.x / KP; r < g_eff * EB; r += rstride) {
    const int i = r % EB;
    if (i >= cnt) continue;
    const uint8_t f = rs.flag[r];
    const double e = (real && f != 2) ? emission_rc(f == 1, rs.x[r], rs.y[r], kc) : 0.0;
    buf[static_cast<size_t>(r) * KP + j] = e;  // r = s*EB + i: buf[s][i][j]
  }
}

// Row renormalisation including the (quad-replicated) tail entries.
template <int NT, int TAIL>
__device__ __forceinline__ void renorm_row_tail(double (&a)[NT][2], double (&at)[TAIL > 0 ? TAIL : 1],
                                                double& rexp) {
  double mx = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(a[nt][0], a[nt][1]));
#pragma unroll
  for (int j = 0; j < TAIL; ++j) mx = fmax(mx, at[j]);
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 2));
  if (mx > 0.0) {
    const int ex = ilogb(mx);
    scale_row<NT>(a, ex);
#pragma unroll
    for (int j = 0; j < TAIL; ++j) at[j] = scale_pow2(at[j], -ex);
    rexp += static_cast<double>(ex);
  }
}

// ---------------------------------------------------------------------------
// Chain kernel: one CTA per (group of G consecutive segments, proposal).
// blockDim.x = 32 * W with 8W >= G*K; warp w owns stacked rows 8w..8w+7.
//
// Head/tail split (TAIL > 0, K = 8*NT + TAIL with TAIL <= 4): the first 8*NT
// states go through the DMMA tiles with no padding at all; the TAIL remaining
// states are carried in registers, replicated in the 4 lanes of each quad,
// and coupled to the head with FP64 FMAs:
//     head' = head * G11 + tail (x) G21        (rank-TAIL update, SIMT)
//     tail' = head . G12 (quad reduction) + tail * G22
// instead of padding K up to the next multiple of 8 (K=25: 18 DMMAs per
// 8-row tile and step instead of 28, ~16 FP64 FMAs per lane extra).
// ---------------------------------------------------------------------------
template <int NT, bool SKIP, int TAIL>
__global__ void __launch_bounds__(chain_max_threads(NT + (TAIL > 0)), chain_min_blocks(NT + (TAIL > 0)))
    chain_f64_kernel(const ChainArgs args) {
  constexpr bool LEAN = chain_lean(NT + (TAIL > 0));
  constexpr int KPE = 8 * (NT + (TAIL > 0 ? 1 : 0));  // padded K: node and emission row width
  constexpr int H = 8 * NT;                            // first tail state
  constexpr int TA = TAIL > 0 ? TAIL : 1;              // array extent
  constexpr int EB = chain_eb(NT + (TAIL > 0));
  const int G = args.G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* bsm = reinterpret_cast<double2*>(smem_raw);               // NT*NT*32 pairs
  double2* g21 = bsm + NT * NT * 32;                                  // [TAIL][NT][4]: G[H+j][8nt+2q+h]
  double2* g12 = g21 + TAIL * NT * 4;                                 // [TAIL][NT][4]: G[8nb+2q+h][H+j]
  double* esm = reinterpret_cast<double*>(g12 + TAIL * NT * 4);      // 2 x G*EB*KPE (double buffer)
  const size_t esm_stride = static_cast<size_t>(G) * EB * KPE;
  double* psm = esm + 2 * esm_stride;                                // 8*KPE emission constants
  double* g22 = psm + 8 * KPE;                                       // TAIL*TAIL
  double* rsm = g22 + TAIL * TAIL;                                   // 8W row exponents
  int64_t* sseg = reinterpret_cast<int64_t*>(rsm + blockDim.x / 4);  // G x (first record, length)
  const RecordStage rstage = record_stage_at(sseg + 2 * G, G, EB);

  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;
  const int64_t seg0 = static_cast<int64_t>(blockIdx.x) * G;
  const int g_eff = static_cast<int>(min(static_cast<int64_t>(G), args.nseg - seg0));

  // This CTA's records: segments seg0 .. seg0+g_eff-1 (contiguous; lengths differ by <= 1,
  // earlier ones longer).
  int64_t first_lo, first_hi, last_lo, last_hi;
  segment_range(args.n, args.nseg, seg0, first_lo, first_hi);
  segment_range(args.n, args.nseg, seg0 + g_eff - 1, last_lo, last_hi);
  const int64_t len_max = first_hi - first_lo, len_min = last_hi - last_lo;

  // My stacked row -> (local segment, state).
  const int row = 8 * warp + g;
  const int s_loc = row / K;
  const int r = row - s_loc * K;
  const bool live = s_loc < g_eff;
  int64_t my_lo = 0, my_hi = 0;
  if (live) segment_range(args.n, args.nseg, seg0 + s_loc, my_lo, my_hi);
  const int64_t my_len = my_hi - my_lo;

  const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
  stage_b_fragments<NT>(bsm, gam, K, K);  // with a tail, only head states are ever indexed
  if (TAIL > 0) {
    for (int idx = threadIdx.x; idx < TAIL * NT * 4; idx += blockDim.x) {
      const int j = idx / (NT * 4), nt = (idx >> 2) % NT, qq = idx & 3;
      const int c0 = 8 * nt + 2 * qq;
      g21[idx] = make_double2(gam[(H + j) * K + c0], gam[(H + j) * K + c0 + 1]);
      g12[idx] = make_double2(gam[c0 * K + H + j], gam[(c0 + 1) * K + H + j]);
    }
    for (int idx = threadIdx.x; idx < TAIL * TAIL; idx += blockDim.x)
      g22[idx] = gam[(H + idx / TA) * K + H + idx % TA];
  }
  if (threadIdx.x < g_eff) {
    int64_t slo, shi;
    segment_range(args.n, args.nseg, seg0 + threadIdx.x, slo, shi);
    sseg[2 * threadIdx.x] = args.lo + slo;
    sseg[2 * threadIdx.x + 1] = shi - slo;
  }
  for (int idx = threadIdx.x; idx < 8 * KPE; idx += blockDim.x) {
    const int f = idx / KPE, j = idx - f * KPE;
    double v = 0.0;
    if (j < K) {
      const double* st = args.P.states;
      if (f < 7) {
        v = st[(static_cast<size_t>(f) * args.B + b) * K + j];
      } else {
        const double ld = st[(static_cast<size_t>(7) * args.B + b) * K + j];
        v = __dsub_rn(args.neg_log_2pi, __dmul_rn(0.5, ld));
      }
    } else if (f == 4 || f == 6) {
      v = 1.0;  // padding states: harmless divisor
    }
    psm[idx] = v;
  }

  double a[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    a[nt][0] = (live && r == 8 * nt + 2 * q) ? 1.0 : 0.0;
    a[nt][1] = (live && r == 8 * nt + 2 * q + 1) ? 1.0 : 0.0;
  }
  double at[TA];
#pragma unroll
  for (int j = 0; j < TA; ++j) at[j] = (TAIL > 0 && live && r == H + j) ? 1.0 : 0.0;
  double rexp = 0.0;
  int since = 0;
  const int period = args.period;
  const double* my_e0 = esm + static_cast<size_t>(live ? s_loc : 0) * EB * KPE;
  __syncthreads();  // constants, segment table and B fragments staged

  // Emission blocks are double-buffered: while a warp runs the DMMA steps of
  // block j it may already be computing block j+1, and warps that finish
  // their share of the emission work early go straight back to the tensor
  // pipe, so the exp/div work overlaps the MMAs of other warps.  One barrier
  // per block.
  const int64_t nblk = (len_max + EB - 1) / EB;
  fill_emission_block<KPE, EB>(args, esm, psm, sseg, 0, len_max, g_eff, rstage);
  __syncthreads();
  // debug trace (tools/f64_trace.cu): lane 0 of every warp of CTA 0 stamps each block
  const bool tr = args.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0;
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t t0 = blk * EB;
    const int cnt = static_cast<int>(len_max - t0 < EB ? len_max - t0 : EB);
    long long s0 = 0, s1 = 0, s2 = 0;
    if (tr) s0 = clock64();
    if (blk + 1 < nblk)
      fill_emission_block<KPE, EB>(args, esm + ((blk + 1) & 1) * esm_stride, psm, sseg, t0 + EB, len_max, g_eff,
                               rstage);
    if (tr) s1 = clock64();
    const double* ebuf = my_e0 + (blk & 1) * esm_stride;
    // Steps where every stacked segment is still running need no predicate.
    const int uniform = static_cast<int>(min(static_cast<int64_t>(cnt), max(len_min - t0, int64_t(0))));
    for (int i = 0; i < cnt; ++i) {
      double c[NT][2];
      tile_product<NT, SKIP, LEAN>(c, a, bsm, lane);
      double ct[TA];
      if (TAIL > 0) {
        // tail' = head . G12 + tail * G22 (uses this step's old head and tail)
#pragma unroll
        for (int j = 0; j < TAIL; ++j) {
          double sacc = 0.0;
#pragma unroll
          for (int nb = 0; nb < NT; ++nb) {
            const double2 co = LEAN ? lds_f64x2(g12 + (j * NT + nb) * 4 + q) : g12[(j * NT + nb) * 4 + q];
            sacc = fma(a[nb][0], co.x, sacc);
            sacc = fma(a[nb][1], co.y, sacc);
          }
          sacc += __shfl_xor_sync(kFull, sacc, 1);
          sacc += __shfl_xor_sync(kFull, sacc, 2);
#pragma unroll
          for (int i2 = 0; i2 < TAIL; ++i2) sacc = fma(at[i2], g22[i2 * TA + j], sacc);
          ct[j] = sacc;
        }
        // head' += tail (x) G21
#pragma unroll
        for (int j = 0; j < TAIL; ++j) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double2 co = LEAN ? lds_f64x2(g21 + (j * NT + nt) * 4 + q) : g21[(j * NT + nt) * 4 + q];
            c[nt][0] = fma(at[j], co.x, c[nt][0]);
            c[nt][1] = fma(at[j], co.y, c[nt][1]);
          }
        }
      }
      const double* erow = ebuf + i * KPE;
      if (i < uniform || t0 + i < my_len) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 ev = *reinterpret_cast<const double2*>(erow + 8 * nt + 2 * q);
          a[nt][0] = c[nt][0] * ev.x;
          a[nt][1] = c[nt][1] * ev.y;
        }
#pragma unroll
        for (int j = 0; j < TAIL; ++j) at[j] = ct[j] * erow[H + j];
      }
      if (++since == period) {
        since = 0;
        renorm_row_tail<NT, TAIL>(a, at, rexp);
      }
    }
    if (tr) s2 = clock64();
    __syncthreads();
    if (tr && blk < 64) {
      long long* o = args.trace + (static_cast<size_t>(warp) * 64 + blk) * 4;
      o[0] = s0;
      o[1] = s1;
      o[2] = s2;
      o[3] = clock64();
    }
  }
  renorm_row_tail<NT, TAIL>(a, at, rexp);

  // Per-segment node exponent E_s = max over the segment's live rows.
  double mx = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(a[nt][0], a[nt][1]));
#pragma unroll
  for (int j = 0; j < TAIL; ++j) mx = fmax(mx, at[j]);
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 2));
  if (q == 0) rsm[row] = (live && mx > 0.0) ? rexp : -INFINITY;
  __syncthreads();
  if (!live) return;
  double E = -INFINITY;
  for (int j = 0; j < K; ++j) E = fmax(E, rsm[s_loc * K + j]);
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg0 + s_loc;
  double* nrow = args.seg_m + node * KPE * KPE + static_cast<size_t>(r) * KPE;
  const bool zero = E == -INFINITY || !(mx > 0.0);
  const int sh = zero ? 0 : static_cast<int>(fmax(rexp - E, -2100.0));  // <= 0
  auto scaled = [&](double v) { return (zero || sh < -2044) ? 0.0 : scale_pow2(v, sh); };
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
    *reinterpret_cast<double2*>(nrow + 8 * nt + 2 * q) = make_double2(scaled(a[nt][0]), scaled(a[nt][1]));
  if (TAIL > 0) {
    // last 8-column tile: tail states then zero padding (2 columns per lane)
    const int c0 = 2 * q;
    double v0 = 0.0, v1 = 0.0;
#pragma unroll
    for (int j = 0; j < TAIL; ++j) {  // static indices only: at[] stays in registers
      if (j == c0) v0 = scaled(at[j]);
      if (j == c0 + 1) v1 = scaled(at[j]);
    }
    *reinterpret_cast<double2*>(nrow + H + c0) = make_double2(v0, v1);
  }
  // Zero the padding rows K..KPE-1 of the node (written by the segment's row-0 quad).
  if (r == 0) {
    for (int pr = K; pr < KPE; ++pr) {
      double* prow = args.seg_m + node * KPE * KPE + static_cast<size_t>(pr) * KPE;
      for (int cc = 2 * q; cc < KPE; cc += 8) *reinterpret_cast<double2*>(prow + cc) = make_double2(0.0, 0.0);
    }
    if (q == 0) args.seg_e[node] = (E == -INFINITY) ? 0.0 : E;
  }
}

// ---------------------------------------------------------------------------
// Fold kernel: one CTA (NT warps) per (group, proposal).  Multiplies the nodes
// of group j = segment_bounds(n_in, n_out)[j] in order, renormalising the
// running product by an exact power of two after each multiply.  With
// finish set (n_out == 1) it returns log(delta' M 1) + e ln 2 instead.
// ---------------------------------------------------------------------------
template <int NT, bool SKIP>
__global__ void __launch_bounds__(NT * 32) fold_kernel(const FoldArgs args) {
  constexpr int KP = NT * 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* bsm = reinterpret_cast<double2*>(smem_raw);
  double* red = reinterpret_cast<double*>(bsm + NT * NT * 32);

  const int grp = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int row = 8 * warp + g;

  int64_t lo, hi;
  segment_range(args.n_in, args.n_out, grp, lo, hi);
  auto node_index = [&](int64_t i) -> int64_t { return i * args.stride_i + b * args.stride_b; };

  double a[NT][2];
  {
    const double* m0 = args.in_m + node_index(lo) * KP * KP + static_cast<size_t>(row) * KP + 2 * q;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const double2 v = *reinterpret_cast<const double2*>(m0 + 8 * nt);
      a[nt][0] = v.x;
      a[nt][1] = v.y;
    }
  }
  double E = args.in_e[node_index(lo)];
  for (int64_t i = lo + 1; i < hi; ++i) {
    __syncthreads();
    stage_b_fragments<NT>(bsm, args.in_m + node_index(i) * KP * KP, KP, KP);
    __syncthreads();
    double c[NT][2];
    tile_product<NT, SKIP>(c, a, bsm, lane);
    E += args.in_e[node_index(i)];
    double mx = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(c[nt][0], c[nt][1]));
    mx = block_max(mx, red, NT);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      a[nt][0] = c[nt][0];
      a[nt][1] = c[nt][1];
    }
    if (mx > 0.0) {
      const int ex = ilogb(mx);
      scale_row<NT>(a, ex);
      E += static_cast<double>(ex);
    }
  }

  if (args.finish) {
    // log(delta' M 1) + E ln 2 ; rows >= K are zero padding.
    double rs = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) rs += a[nt][0] + a[nt][1];
    rs += __shfl_xor_sync(kFull, rs, 1);
    rs += __shfl_xor_sync(kFull, rs, 2);
    const double w = (row < args.K && q == 0) ? args.delta[static_cast<size_t>(b) * args.K + row] * rs : 0.0;
    const double s = block_sum(w, red, NT);
    if (threadIdx.x == 0) {
      const bool ok = s > 0.0 && isfinite(s);
      args.loglik[b] = ok ? log(s) + E * 0.69314718055994530942 : -INFINITY;
      args.status[b] = ok ? 0 : 2;
    }
  } else {
    double* out = args.out_m + (static_cast<size_t>(b) * args.n_out + grp) * KP * KP +
                  static_cast<size_t>(row) * KP + 2 * q;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) *reinterpret_cast<double2*>(out + 8 * nt) = make_double2(a[nt][0], a[nt][1]);
    if (threadIdx.x == 0) args.out_e[static_cast<size_t>(b) * args.n_out + grp] = E;
  }
}

// ---------------------------------------------------------------------------
// Whole segment tree in one launch.  Level-1 CTAs fold radix-R groups of the
// level-0 nodes; each finished node bumps its parent's arrival counter and
// the last child to arrive carries on with the parent group (device-scope
// fence + atomic, nodes of other CTAs read with ld.global.cg).  The CTA that
// completes the root evaluates log(delta' M 1) + e ln 2 (or writes the root
// node for a multi-GPU shard).  No per-level launch gaps; counters are reset
// by their last user, so they are zero again when the kernel ends.
// ---------------------------------------------------------------------------
constexpr int kTreeMaxLevels = 12;

struct TreeArgs {
  const double* in_m;   // level-0 node (b, i) at in_m + i*m_stride_i + b*m_stride_b (doubles)
  const double* in_e;   //          exponent at in_e[i*e_stride_i + b*e_stride_b]
  int64_t m_stride_i;
  int64_t m_stride_b;
  int64_t e_stride_i;
  int64_t e_stride_b;
  int radix;
  int levels;                         // levels above level 0; count[levels] == 1
  int64_t count[kTreeMaxLevels + 1];  // nodes per proposal at each level (count[0] = level-0 nodes)
  int64_t off[kTreeMaxLevels + 1];    // first scratch node of level l (levels 1..levels-1), layout [B][count]
  int64_t cnt_off[kTreeMaxLevels + 1];  // first counter of level l (levels 2..levels), layout [B][count]
  double* scratch_m;
  double* scratch_e;
  unsigned* counters;
  int K;
  int B;
  int finish;
  const double* delta;
  double* loglik;
  int32_t* status;
  double* out_m;  // root nodes [B] when !finish
  double* out_e;
};

__device__ __forceinline__ double2 ldcg_f64x2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

// Warp groups per tree CTA: each folds up to kTreeGroupRadix children in
// order, then group 0 multiplies by group 1's partial.  Two groups (radix 8:
// four dependent products per level, half the levels) where the products are
// short and the level latency is arrival + loads (padded K <= 32: the tree
// 15-25% faster); one group (radix 4) for wide rows, whose products already
// fill the SM's DMMA pipe.
constexpr int kTreeGroupRadix = 4;
__host__ __device__ constexpr int tree_groups(int nt) { return nt <= 4 ? 2 : 1; }
__host__ __device__ constexpr int tree_radix(int nt) { return tree_groups(nt) * kTreeGroupRadix; }

__host__ __device__ constexpr size_t tree_smem_bytes(int nt) {
  return static_cast<size_t>(tree_groups(nt) + 1) * nt * nt * 32 * 16 +  // B fragments per group + group 1's partial
         static_cast<size_t>(tree_groups(nt)) * nt * 8 + 16;            // per-warp maxima, partial exponent
}

template <int NT, bool SKIP>
__global__ void __launch_bounds__(tree_groups(NT) * NT * 32) tree_fold_kernel(const TreeArgs args) {
  constexpr int KP = NT * 8;
  constexpr int GT = NT * 32;
  constexpr int kTreeGroups = tree_groups(NT);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / NT, wg = warp - grp * NT;
  double2* bsm = reinterpret_cast<double2*>(smem_raw) + grp * NT * NT * 32;        // this group's B fragments
  double2* psm = reinterpret_cast<double2*>(smem_raw) + kTreeGroups * NT * NT * 32;  // group 1's partial (B frags)
  double* red_all = reinterpret_cast<double*>(psm + NT * NT * 32);
  double* red = red_all + grp * NT;
  double* pexp = red_all + kTreeGroups * NT;
  __shared__ int s_last;

  const int b = blockIdx.y;
  const int g = lane >> 2, q = lane & 3;
  const int row = 8 * wg + g;
  const int R = args.radix;  // == tree_radix(NT)
  const int bar = 1 + grp;
  auto gsync = [&]() { asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(GT) : "memory"); };
  // max over the group (all its threads get it)
  auto group_max = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    gsync();
    if (lane == 0) red[wg] = v;
    gsync();
    double r = red[0];
    for (int w = 1; w < NT; ++w) r = fmax(r, red[w]);
    return r;
  };

  int level = 1;
  int64_t j = blockIdx.x;
  for (;;) {
    // children of node j at `level`: nodes [j*R, min((j+1)*R, count[level-1])) of level-1;
    // group gi folds [c_lo + 4 gi, ...) in order
    const int64_t c_lo = j * R;
    const int64_t c_end = min(c_lo + R, args.count[level - 1]);
    const int64_t g_lo = c_lo + static_cast<int64_t>(kTreeGroupRadix) * grp;  // R == kTreeGroups * kTreeGroupRadix
    const int64_t g_hi = min(g_lo + kTreeGroupRadix, c_end);
    const bool active = g_lo < g_hi;
    const bool from_scratch = level >= 2;
    auto child_m = [&](int64_t i) -> const double* {
      return from_scratch ? args.scratch_m + (args.off[level - 1] + b * args.count[level - 1] + i) * KP * KP
                          : args.in_m + i * args.m_stride_i + b * args.m_stride_b;
    };
    auto child_e = [&](int64_t i) -> double {
      return from_scratch ? __ldcg(args.scratch_e + args.off[level - 1] + b * args.count[level - 1] + i)
                          : args.in_e[i * args.e_stride_i + b * args.e_stride_b];
    };
    double a[NT][2];
    double E = 0.0;
    if (active) {
      {
        const double* m0 = child_m(g_lo) + static_cast<size_t>(row) * KP + 2 * q;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 v = ldcg_f64x2(m0 + 8 * nt);
          a[nt][0] = v.x;
          a[nt][1] = v.y;
        }
      }
      E = child_e(g_lo);
      // The group's remaining children (at most kTreeGroupRadix - 1) are all
      // fetched into registers at once (NT B-fragment pairs per thread and
      // child, GT threads per group): one memory latency per level, not one
      // per child.
      constexpr int NPF = kTreeGroupRadix - 1;
      double2 pf[NPF][NT];
      double pe[NPF];
#pragma unroll
      for (int v = 0; v < NPF; ++v) {
        if (g_lo + 1 + v < g_hi) {
          const double* m = child_m(g_lo + 1 + v);
#pragma unroll
          for (int u = 0; u < NT; ++u) {
            const int idx = (threadIdx.x - grp * GT) + u * GT;
            const int l = idx & 31, pair = idx >> 5;
            const int nb = pair % NT, nt = pair / NT;
            const int k0 = 8 * nb + 2 * (l & 3), col = 8 * nt + (l >> 2);
            pf[v][u] = make_double2(__ldcg(m + k0 * KP + col), __ldcg(m + (k0 + 1) * KP + col));
          }
          pe[v] = child_e(g_lo + 1 + v);
        }
      }
#pragma unroll
      for (int v = 0; v < NPF; ++v) {
        if (g_lo + 1 + v >= g_hi) break;
        gsync();
#pragma unroll
        for (int u = 0; u < NT; ++u) bsm[(threadIdx.x - grp * GT) + u * GT] = pf[v][u];
        gsync();
        double c[NT][2];
        tile_product<NT, SKIP>(c, a, bsm, lane);
        E += pe[v];
        double mx = 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(c[nt][0], c[nt][1]));
        mx = group_max(mx);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          a[nt][0] = c[nt][0];
          a[nt][1] = c[nt][1];
        }
        if (mx > 0.0) {
          const int ex = ilogb(mx);
          scale_row<NT>(a, ex);
          E += static_cast<double>(ex);
        }
      }
      if (grp == 1) {  // publish the partial as B fragments: element (row, col) -> pair (col/8, row/8)
        double* pd = reinterpret_cast<double*>(psm);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = 8 * nt + 2 * q + h;
            pd[2 * (((col >> 3) * NT + (row >> 3)) * 32 + ((col & 7) << 2) + ((row & 7) >> 1)) + (row & 1)] = a[nt][h];
          }
        if (threadIdx.x == GT) *pexp = E;
      }
    }
    __syncthreads();
    const bool two = kTreeGroups > 1 && c_lo + kTreeGroupRadix < c_end;  // group 1 had children
    if (grp == 0 && two) {
      double c[NT][2];
      tile_product<NT, SKIP>(c, a, psm, lane);
      E += *pexp;
      double mx = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(c[nt][0], c[nt][1]));
      mx = group_max(mx);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        a[nt][0] = c[nt][0];
        a[nt][1] = c[nt][1];
      }
      if (mx > 0.0) {
        const int ex = ilogb(mx);
        scale_row<NT>(a, ex);
        E += static_cast<double>(ex);
      }
    }

    if (level == args.levels) {  // root (group 0)
      if (grp == 0) {
        if (args.finish) {
          double rs = 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) rs += a[nt][0] + a[nt][1];
          rs += __shfl_xor_sync(kFull, rs, 1);
          rs += __shfl_xor_sync(kFull, rs, 2);
          double w = (row < args.K && q == 0) ? args.delta[static_cast<size_t>(b) * args.K + row] * rs : 0.0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(kFull, w, o);
          gsync();
          if (lane == 0) red[wg] = w;
          gsync();
          if (threadIdx.x == 0) {
            double s = red[0];
            for (int w2 = 1; w2 < NT; ++w2) s += red[w2];
            const bool ok = s > 0.0 && isfinite(s);
            args.loglik[b] = ok ? log(s) + E * 0.69314718055994530942 : -INFINITY;
            args.status[b] = ok ? 0 : 2;
          }
        } else {
          double* out = args.out_m + static_cast<size_t>(b) * KP * KP + static_cast<size_t>(row) * KP + 2 * q;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            *reinterpret_cast<double2*>(out + 8 * nt) = make_double2(a[nt][0], a[nt][1]);
          if (threadIdx.x == 0) args.out_e[b] = E;
        }
      }
      return;
    }

    // store node j of `level` (group 0), then arrive at the parent's counter
    if (grp == 0) {
      const int64_t slot = args.off[level] + b * args.count[level] + j;
      double* out = args.scratch_m + slot * KP * KP + static_cast<size_t>(row) * KP + 2 * q;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) *reinterpret_cast<double2*>(out + 8 * nt) = make_double2(a[nt][0], a[nt][1]);
      if (threadIdx.x == 0) args.scratch_e[slot] = E;
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t parent = j / R;
      const int64_t nchild = min(static_cast<int64_t>(R), args.count[level] - parent * R);
      unsigned* ctr = args.counters + args.cnt_off[level + 1] + b * args.count[level + 1] + parent;
      const unsigned prev = atomicAdd(ctr, 1u);
      const bool last = prev + 1 == static_cast<unsigned>(nchild);
      if (last) *ctr = 0u;  // every child has arrived: reset for the next launch
      s_last = last ? 1 : 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    j /= R;
    ++level;
  }
}

// ---------------------------------------------------------------------------
// FP32 chain (EngineConfig(precision="float32"), reference engine.py:331-333:
// factor products in float32 storage, emission table cast to float32, logs in
// float64).  SIMT: one thread owns one stacked row of the running product, so
// the per-row renormalisation needs no communication; Gamma (float32) is read
// from shared memory as broadcast float4 rows, the thread's row from its own
// conflict-free shared-memory slot.  Renormalises every step by an exact power
// of two (the FP32 range is too narrow to skip steps safely); the node is
// emitted in the FP64 node format, so the fold tree is shared with the FP64
// path (the reference also combines in float64, engine.py:307-318).
// ---------------------------------------------------------------------------
constexpr int kEmissionBlock32 = 16;

__host__ __device__ constexpr int chain32_max_threads(int nt) {
  return nt <= 4 ? 1024 : (nt <= 6 ? 512 : 384);
}

__host__ __device__ constexpr size_t chain32_smem_bytes(int nt, int G, int threads) {
  return static_cast<size_t>(nt * 8) * (nt * 8) * 4 +                        // Gamma (f32)
         static_cast<size_t>(2) * G * kEmissionBlock32 * nt * 8 * 4 +        // emission blocks (x2)
         static_cast<size_t>(8) * nt * 8 * 8 +                               // emission constants
         static_cast<size_t>(threads) * 8 +                                  // row exponents
         static_cast<size_t>(16) * G +                                       // segment table
         static_cast<size_t>(threads) * (nt * 8 + 1) * 4 +                   // rows (f32)
         record_stage_bytes(G, kEmissionBlock32);                            // staged records
}

__device__ __forceinline__ float pow2f_normal(int n) {  // n in [-126, 127]
  return __int_as_float((n + 127) << 23);
}

template <int KP>
__device__ __forceinline__ void fill_emission_block32(const ChainArgs& args, float* buf, const double* psm,
                                                      const int64_t* sseg, int64_t t0, int64_t len_max,
                                                      int g_eff, RecordStage rs) {
  constexpr int EB = kEmissionBlock32;
  const int cnt = static_cast<int>(len_max - t0 < EB ? len_max - t0 : EB);
  stage_records<EB, false>(args, rs, sseg, t0, cnt, g_eff, len_max);
  const int j = threadIdx.x % KP;
  const int rstride = blockDim.x / KP;
  if (static_cast<int>(threadIdx.x) >= rstride * KP) return;
  const bool real = j < args.K;
  const StateConsts kc = load_state_consts(psm + j, KP);
  for (int r = threadIdx.x / KP; r < g_eff * EB; r += rstride) {
    if (r % EB >= cnt) continue;
    const uint8_t f = rs.flag[r];
    buf[static_cast<size_t>(r) * KP + j] =
        (real && f != 2) ? static_cast<float>(emission_rc(f == 1, rs.x[r], rs.y[r], kc)) : 0.0f;
  }
}

template <int NT>
__global__ void __launch_bounds__(chain32_max_threads(NT)) chain_f32_kernel(const ChainArgs args) {
  constexpr int KP = NT * 8;
  constexpr int AS = KP + 1;  // odd row stride: conflict-free per-thread rows
  constexpr int EB = kEmissionBlock32;
  const int G = args.G;
  const int threads = blockDim.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* gsm = reinterpret_cast<float*>(smem_raw);                       // KP*KP
  float* esm = gsm + KP * KP;                                             // 2 x G*EB*KP
  const size_t esm_stride = static_cast<size_t>(G) * EB * KP;
  double* psm = reinterpret_cast<double*>(esm + 2 * esm_stride);          // 8*KP
  double* rsm = psm + 8 * KP;                                             // threads
  int64_t* sseg = reinterpret_cast<int64_t*>(rsm + threads);             // 2G
  float* rows = reinterpret_cast<float*>(sseg + 2 * G);                   // threads*AS
  const RecordStage rstage = record_stage_at(rows + static_cast<size_t>(threads) * AS, G, EB);

  const int b = blockIdx.y;
  const int K = args.K;
  const int64_t seg0 = static_cast<int64_t>(blockIdx.x) * G;
  const int g_eff = static_cast<int>(min(static_cast<int64_t>(G), args.nseg - seg0));
  int64_t first_lo, first_hi;
  segment_range(args.n, args.nseg, seg0, first_lo, first_hi);
  const int64_t len_max = first_hi - first_lo;

  const int row = threadIdx.x;
  const int s_loc = row / K;
  const int r = row - s_loc * K;
  const bool live = s_loc < g_eff;
  int64_t my_lo = 0, my_hi = 0;
  if (live) segment_range(args.n, args.nseg, seg0 + s_loc, my_lo, my_hi);
  const int64_t my_len = my_hi - my_lo;

  const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
  for (int idx = threadIdx.x; idx < KP * KP; idx += threads) {
    const int i = idx / KP, j = idx - i * KP;
    gsm[idx] = (i < K && j < K) ? static_cast<float>(gam[i * K + j]) : 0.0f;
  }
  if (threadIdx.x < g_eff) {
    int64_t slo, shi;
    segment_range(args.n, args.nseg, seg0 + threadIdx.x, slo, shi);
    sseg[2 * threadIdx.x] = args.lo + slo;
    sseg[2 * threadIdx.x + 1] = shi - slo;
  }
  for (int idx = threadIdx.x; idx < 8 * KP; idx += threads) {
    const int f = idx / KP, j = idx - f * KP;
    double v = (f == 4 || f == 6) ? 1.0 : 0.0;
    if (j < K) {
      const double* st = args.P.states;
      v = f < 7 ? st[(static_cast<size_t>(f) * args.B + b) * K + j]
                : __dsub_rn(args.neg_log_2pi, __dmul_rn(0.5, st[(static_cast<size_t>(7) * args.B + b) * K + j]));
    }
    psm[idx] = v;
  }
  float* my_row = rows + static_cast<size_t>(row) * AS;
  for (int c = 0; c < KP; ++c) my_row[c] = (live && c == r) ? 1.0f : 0.0f;
  double rexp = 0.0;
  float acc[KP];
  const float* my_e = esm + static_cast<size_t>(live ? s_loc : 0) * EB * KP;
  __syncthreads();

  const int64_t nblk = (len_max + EB - 1) / EB;
  fill_emission_block32<KP>(args, esm, psm, sseg, 0, len_max, g_eff, rstage);
  __syncthreads();
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t t0 = blk * EB;
    const int cnt = static_cast<int>(len_max - t0 < EB ? len_max - t0 : EB);
    if (blk + 1 < nblk)
      fill_emission_block32<KP>(args, esm + ((blk + 1) & 1) * esm_stride, psm, sseg, t0 + EB, len_max, g_eff,
                                rstage);
    const float* ebuf = my_e + (blk & 1) * esm_stride;
    for (int i = 0; i < cnt; ++i) {
      if (!live || t0 + i >= my_len) continue;
#pragma unroll
      for (int c = 0; c < KP; ++c) acc[c] = 0.0f;
#pragma unroll 2
      for (int k = 0; k < KP; ++k) {
        const float a = my_row[k];
        const float4* g4 = reinterpret_cast<const float4*>(gsm + k * KP);
#pragma unroll
        for (int c4 = 0; c4 < KP / 4; ++c4) {
          const float4 gv = g4[c4];
          acc[4 * c4 + 0] = fmaf(a, gv.x, acc[4 * c4 + 0]);
          acc[4 * c4 + 1] = fmaf(a, gv.y, acc[4 * c4 + 1]);
          acc[4 * c4 + 2] = fmaf(a, gv.z, acc[4 * c4 + 2]);
          acc[4 * c4 + 3] = fmaf(a, gv.w, acc[4 * c4 + 3]);
        }
      }
      const float4* e4 = reinterpret_cast<const float4*>(ebuf + i * KP);
      float mx = 0.0f;
#pragma unroll
      for (int c4 = 0; c4 < KP / 4; ++c4) {
        const float4 ev = e4[c4];
        acc[4 * c4 + 0] *= ev.x;
        acc[4 * c4 + 1] *= ev.y;
        acc[4 * c4 + 2] *= ev.z;
        acc[4 * c4 + 3] *= ev.w;
        mx = fmaxf(mx, fmaxf(fmaxf(acc[4 * c4 + 0], acc[4 * c4 + 1]), fmaxf(acc[4 * c4 + 2], acc[4 * c4 + 3])));
      }
      if (mx > 0.0f) {
        const int ex = ilogbf(mx);
        if (ex >= -126 && ex <= 126) {
          const float sc = pow2f_normal(-ex);
#pragma unroll
          for (int c = 0; c < KP; ++c) acc[c] *= sc;
        } else {
#pragma unroll
          for (int c = 0; c < KP; ++c) acc[c] = scalbnf(acc[c], -ex);
        }
        rexp += static_cast<double>(ex);
      }
#pragma unroll
      for (int c = 0; c < KP; ++c) my_row[c] = acc[c];
    }
    __syncthreads();
  }

  // Node (FP64 format): per-segment exponent E = max over live rows.
  float mx = 0.0f;
  for (int c = 0; c < KP; ++c) mx = fmaxf(mx, my_row[c]);
  rsm[row] = (live && mx > 0.0f) ? rexp : -INFINITY;
  __syncthreads();
  if (!live) return;
  double E = -INFINITY;
  for (int j = 0; j < K; ++j) E = fmax(E, rsm[s_loc * K + j]);
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg0 + s_loc;
  double* out = args.seg_m + node * KP * KP + static_cast<size_t>(r) * KP;
  const bool zero = (E == -INFINITY) || !(mx > 0.0f);
  const int sh = zero ? 0 : static_cast<int>(fmax(rexp - E, -2100.0));
  for (int c = 0; c < KP; ++c)
    out[c] = (zero || sh < -2044) ? 0.0 : scale_pow2(static_cast<double>(my_row[c]), sh);
  if (r == 0) {
    for (int pr = K; pr < KP; ++pr)
      for (int c = 0; c < KP; ++c) args.seg_m[node * KP * KP + static_cast<size_t>(pr) * KP + c] = 0.0;
    args.seg_e[node] = (E == -INFINITY) ? 0.0 : E;
  }
}

// Emission table for records [lo, lo+n) of parameter set 0 (reference
// _emission_columns, core.py:235-260); explicit-table API.  CHAIN: the
// arithmetic of the chain kernels' emission stage instead (emission_rc from
// register constants, the same device function runs_emissions and the
// record-by-record chain call) -- the diagnostic entry that lets the tests
// check the hot path's emission values directly.
template <bool CHAIN>
__global__ void emission_table_kernel(const uint8_t* __restrict__ present, const double* __restrict__ lon,
                                      const double* __restrict__ lat, int64_t lo, int64_t n, int K,
                                      const double* __restrict__ states, int B, double neg_log_2pi,
                                      double* __restrict__ out) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * K) return;
  const int64_t i = idx / K;
  const int j = static_cast<int>(idx - i * K);
  const int64_t t = lo + i;
  double pj[8 * 1];
  for (int f = 0; f < 7; ++f) pj[f] = states[(static_cast<size_t>(f) * B) * K + j];
  pj[7] = __dsub_rn(neg_log_2pi, __dmul_rn(0.5, states[(static_cast<size_t>(7) * B) * K + j]));
  if (CHAIN) {
    const StateConsts kc = load_state_consts(pj, 1);
    out[idx] = emission_rc(present[t] != 0, lon[t], lat[t], kc);
  } else {
    out[idx] = emission(present[t] != 0, lon[t], lat[t], pj, 1);
  }
}

}  // namespace thmm
