// thmm_tc.cuh -- TF32 tensor-core (tcgen05 / TMEM) chain kernel for the
// precision study of BASELINE.json configs[3] (FP64 vs FP32/TF32).
//
// Same recursion as chain_f64_kernel (reference engine.py:133-179): every
// stacked row of a segment product runs  row <- (row . Gamma) o e_t,  with
// the reference's float32 semantics (engine.py:331-333: emission evaluated in
// FP64 and stored as float32, products in float32, log-scales in float64).
// The product runs on the 5th-generation tensor cores:
//
//   * A CTA owns T tiles of 128 stacked rows (G whole segments, rows of one
//     segment never straddle CTAs).  Tile w is driven by warpgroup w: thread
//     (w, l) owns row l of the tile, which is TMEM lane l of the tile's
//     accumulator, so the per-row renormalisation is thread-local.
//   * Per step and tile one elected thread issues
//         D[128 x NP] (TMEM, f32) = A[128 x KP] (TMEM, tf32) . B[KP x NP] (smem, tf32)
//     as KP/8 tcgen05.mma.kind::tf32 instructions with A read from TMEM
//     (the previous step's rows, written back with tcgen05.st) and B = Gamma
//     in the canonical K-major no-swizzle core-matrix layout, committed to
//     the tile's mbarrier.  The warpgroup waits, tcgen05.ld's its rows,
//     multiplies by the emission row, rescales by an exact power of two and
//     stores the next A.  The T warpgroups interleave, so the tensor pipe
//     runs one tile's MMAs while the others are in their epilogues.
//   * x3 ("tf32x3"): rows and Gamma are split hi + lo (both tf32) and each
//     step is  Alo.Bhi + Ahi.Blo + Ahi.Bhi  -- ~FP32-accurate products at a
//     third of the TF32 rate.  "tf32x2" keeps only Gamma's split
//     (Ahi.Blo + Ahi.Bhi): the fixed transition matrix is exact to ~2^-22
//     and only the rows are rounded to tf32, afresh on every step.  Plain
//     "tf32" uses Ahi.Bhi only (10-bit mantissa operands).
//
// Nodes are written in the FP64 node format, so the segment tree and the
// multi-GPU combine are shared with the FP64 path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "thmm_kernels.cuh"

namespace thmm {

constexpr int kTcRows = 128;  // rows per tile (UMMA M)

__host__ __device__ constexpr int tc_np(int K) { return ((K + 15) / 16) * 16; }  // UMMA N (multiple of 16)
__host__ __device__ constexpr int tc_kp(int K) { return ((K + 7) / 8) * 8; }     // contraction, 8 per MMA
__host__ __device__ constexpr int tc_cols(int np, int kp, bool x3) { return np + kp * (x3 ? 2 : 1); }
__host__ __device__ constexpr int tc_min2(int a, int b) { return a < b ? a : b; }
// Threads per tile: 128 rows x H column slices (H = 2 splits each row's
// epilogue over two warps of the same TMEM lane quarter).
__host__ __device__ constexpr int tc_tile_threads(int h) { return kTcRows * h; }
// Tiles per CTA: TMEM (1x columns), 1024 threads, and the register budget of
// a row slice of NP/H floats (1 CTA per SM).
__host__ __device__ constexpr int tc_max_tiles(int np, int kp, int h) {
  return tc_min2(tc_min2(8, 512 / tc_cols(np, kp, false)),
                 tc_min2(1024 / tc_tile_threads(h),
                         np / h <= 16 ? 8 : (np / h <= 32 ? 6 : (np / h <= 48 ? 5 : (np / h <= 64 ? 4 : 3)))));
}
__host__ __device__ constexpr int tc_max_threads(int np, int kp, int h) {
  return tc_tile_threads(h) * tc_max_tiles(np, kp, h);
}

__host__ __device__ constexpr size_t tc_align(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ constexpr size_t chain_tc_smem_bytes(int np, int kp, int G, int T, int h = 1) {
  return tc_align(static_cast<size_t>(2) * np * kp * 4, 16) +                        // B hi | lo (tf32)
         tc_align(static_cast<size_t>(2) * G * kEmissionBlock32 * np * 4, 16) +      // emission blocks (x2)
         static_cast<size_t>(8) * np * 8 +                                           // emission constants
         static_cast<size_t>(T) * kTcRows * 8 +                                      // row exponents
         static_cast<size_t>(2) * T * h * kTcRows * 4 +                              // row-max slices (x2)
         static_cast<size_t>(16) * G +                                               // segment table
         static_cast<size_t>(8) * T + 16 +                                           // mbarriers, TMEM slot
         record_stage_bytes(G, kEmissionBlock32);                                    // staged records
}

// ---- PTX wrappers ----------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x));
  return u;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem desc]
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

#define THMM_R16(r, o)                                                                                          \
  "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]),            \
      "=r"(r[o + 6]), "=r"(r[o + 7]), "=r"(r[o + 8]), "=r"(r[o + 9]), "=r"(r[o + 10]), "=r"(r[o + 11]),      \
      "=r"(r[o + 12]), "=r"(r[o + 13]), "=r"(r[o + 14]), "=r"(r[o + 15])
#define THMM_W16(r, o)                                                                                          \
  "r"(r[o + 0]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3]), "r"(r[o + 4]), "r"(r[o + 5]), "r"(r[o + 6]),   \
      "r"(r[o + 7]), "r"(r[o + 8]), "r"(r[o + 9]), "r"(r[o + 10]), "r"(r[o + 11]), "r"(r[o + 12]),            \
      "r"(r[o + 13]), "r"(r[o + 14]), "r"(r[o + 15])

// N consecutive 32-bit TMEM columns of this thread's lane (N multiple of 8).
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t (&r)[N], uint32_t addr) {
  static_assert(N % 8 == 0, "columns in multiples of 8");
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : THMM_R16(r, c)
        : "r"(addr + c));
  if constexpr (N % 16 == 8) {
    constexpr int c = N - 8;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                   "=r"(r[c + 6]), "=r"(r[c + 7])
                 : "r"(addr + c));
  }
}

// Waits for this thread's tcgen05.ld's; the register pass-through keeps the
// compiler from using r[] before the wait.
template <int N>
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[N]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int c = 0; c < N; ++c) asm volatile("" : "+r"(r[c]));
}

template <int N>
__device__ __forceinline__ void tmem_st(uint32_t addr, const uint32_t (&r)[N]) {
  static_assert(N % 8 == 0, "columns in multiples of 8");
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16)
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
            addr + c),
        THMM_W16(r, c)
        : "memory");
  if constexpr (N % 16 == 8) {
    constexpr int c = N - 8;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(addr + c),
                 "r"(r[c]), "r"(r[c + 1]), "r"(r[c + 2]), "r"(r[c + 3]), "r"(r[c + 4]), "r"(r[c + 5]),
                 "r"(r[c + 6]), "r"(r[c + 7])
                 : "memory");
  }
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, no swizzle: core matrices of
// 8 rows x 16 bytes; LBO = byte step between the two K core matrices of one
// MMA, SBO = byte step between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_kmajor(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

// Instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M = 128, N = np.
__host__ __device__ constexpr uint32_t tc_idesc(int np) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(np >> 3) << 17) |
         (static_cast<uint32_t>(kTcRows >> 4) << 24);
}

// Emission block [t0, t0 + EB) of the CTA's G segments, END-aligned: segment
// s (length len_s, off_s = len_max - len_s in {0, 1}) consumes record
// start_s + t - off_s at CTA step t, so every segment of the CTA finishes on
// the same step (the one-record-shorter segments idle on step 0 instead).
// Values: FP64 emission (reference core.py:255-258) stored as float32, the
// reference's float32 semantics (engine.py:331-333).
template <int NP>
__device__ __noinline__ void fill_emission_tc(const ChainArgs& args, float* buf, const double* psm,
                                              const int64_t* sseg, int64_t t0, int64_t len_max, int g_eff,
                                              RecordStage rs) {
  constexpr int EB = kEmissionBlock32;
  const int cnt = static_cast<int>(len_max - t0 < EB ? len_max - t0 : EB);
  stage_records<EB, true>(args, rs, sseg, t0, cnt, g_eff, len_max);
  const int j = threadIdx.x % NP;
  const int rstride = blockDim.x / NP;
  if (static_cast<int>(threadIdx.x) >= rstride * NP) return;
  const bool real = j < args.K;
  const StateConsts kc = load_state_consts(psm + j, NP);
  for (int r = threadIdx.x / NP; r < g_eff * EB; r += rstride) {
    if (r % EB >= cnt) continue;
    const uint8_t f = rs.flag[r];
    buf[static_cast<size_t>(r) * NP + j] =
        (real && f != 2) ? static_cast<float>(emission_rc(f == 1, rs.x[r], rs.y[r], kc)) : 0.0f;
  }
}

// ---------------------------------------------------------------------------
// Chain kernel: one CTA per (group of G consecutive segments, proposal);
// blockDim = 128 T, 128 T >= G K.
//
// Scaling is applied one step late: the rows stored as the next A operand
// are  w = (D o e_t) * 2^-s  with s the exponent of the previous step's row
// max (exact powers of two; the row exponent accumulates s), so one pass
// over the accumulator columns computes, rescales and stores the row and no
// copy of the row is kept in registers across steps.
// ---------------------------------------------------------------------------
template <int NP, int KP, int H>
__global__ void __launch_bounds__(tc_max_threads(NP, KP, H), 1) chain_tc_kernel(const ChainArgs args) {
  constexpr int EB = kEmissionBlock32;
  constexpr int NK = KP / 8;                   // MMAs per product
  constexpr int NPH = NP / H;                  // accumulator columns per thread
  constexpr int TPT = tc_tile_threads(H);      // threads per tile
  static_assert(NPH % 8 == 0, "column slices in multiples of 8");
  constexpr uint32_t LBO = 128, SBO = KP / 4 * 128;
  const bool x3 = args.x3 == 1;   // split rows (A_lo stored) and Gamma
  const bool blo_pass = args.x3 != 0;  // Ahi.Blo pass (tf32x3, tf32x2)
  const int T = blockDim.x / TPT;
  const int G = args.G;
  const int K = args.K;
  const int cols_wg = tc_cols(NP, KP, x3);

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bhi = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* blo = bhi + NP * KP;
  float* esm = reinterpret_cast<float*>(smem_raw + tc_align(static_cast<size_t>(2) * NP * KP * 4, 16));
  const size_t esm_stride = static_cast<size_t>(G) * EB * NP;
  double* psm = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(esm) +
                                          tc_align(2 * esm_stride * sizeof(float), 16));
  double* rsm = psm + 8 * NP;
  float* mxs = reinterpret_cast<float*>(rsm + T * kTcRows);  // [2][T][H][128] row-max slices
  int64_t* sseg = reinterpret_cast<int64_t*>(mxs + 2 * T * H * kTcRows);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sseg + 2 * G);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + T);
  const RecordStage rstage = record_stage_at(tslot + 4, G, EB);

  const int b = blockIdx.y;
  const int tid = threadIdx.x;
  const int wg = tid / TPT, lw = tid % TPT;
  const int wq = (lw >> 5) & 3;        // TMEM lane quarter (= warp id % 4)
  const int hh = (lw >> 5) >> 2;       // column slice
  const int lr = wq * 32 + (lw & 31);  // row of the tile = TMEM lane
  const int c0 = hh * NPH;             // first accumulator column of this thread
  const int64_t seg0 = static_cast<int64_t>(blockIdx.x) * G;
  const int g_eff = static_cast<int>(min(static_cast<int64_t>(G), args.nseg - seg0));
  int64_t first_lo, first_hi;
  segment_range(args.n, args.nseg, seg0, first_lo, first_hi);
  const int64_t len_max = first_hi - first_lo;

  const int row = wg * kTcRows + lr;
  const int s_loc = row / K;
  const int r = row - s_loc * K;
  const bool live = s_loc < g_eff;
  int64_t my_lo = 0, my_hi = 0;
  if (live) segment_range(args.n, args.nseg, seg0 + s_loc, my_lo, my_hi);
  const int64_t my_off = live ? len_max - (my_hi - my_lo) : 0;  // idle steps at the start (0 or 1)

  // B = Gamma as an NP x KP K-major operand: B[n][k] = Gamma[k][n], split hi + lo.
  const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
  for (int idx = tid; idx < NP * KP; idx += blockDim.x) {
    const int n = idx / KP, k = idx - n * KP;
    const double gv = (n < K && k < K) ? gam[k * K + n] : 0.0;
    const uint32_t hi = tf32_rna(static_cast<float>(gv));
    const uint32_t lo = tf32_rna(static_cast<float>(gv - static_cast<double>(__uint_as_float(hi))));
    const int off = ((n >> 3) * (KP / 4) + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3);
    bhi[off] = hi;
    blo[off] = lo;
  }
  if (tid < g_eff) {
    int64_t slo, shi;
    segment_range(args.n, args.nseg, seg0 + tid, slo, shi);
    sseg[2 * tid] = args.lo + slo;
    sseg[2 * tid + 1] = shi - slo;
  }
  for (int idx = tid; idx < 8 * NP; idx += blockDim.x) {
    const int f = idx / NP, j = idx - f * NP;
    double v = (f == 4 || f == 6) ? 1.0 : 0.0;
    if (j < K) {
      const double* st = args.P.states;
      v = f < 7 ? st[(static_cast<size_t>(f) * args.B + b) * K + j]
                : __dsub_rn(args.neg_log_2pi, __dmul_rn(0.5, st[(static_cast<size_t>(7) * args.B + b) * K + j]));
    }
    psm[idx] = v;
  }
  if (tid == 0) {
    for (int w = 0; w < T; ++w) mbar_init(&mbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // TMEM: T tiles x (D | A_hi | A_lo) columns, power of two >= 32.
  uint32_t ncols = 32;
  while (ncols < static_cast<uint32_t>(T * cols_wg)) ncols <<= 1;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
  const uint32_t col_d = tbase + wg * cols_wg;
  const uint32_t col_ahi = col_d + NP, col_alo = col_ahi + KP;
  const uint64_t desc_hi = smem_desc_kmajor(smem_u32(bhi), LBO, SBO);
  const uint64_t desc_lo = smem_desc_kmajor(smem_u32(blo), LBO, SBO);
  constexpr uint32_t idesc = tc_idesc(NP);
  uint64_t* my_bar = &mbar[wg];
  const int bar_id = 1 + wg;

  auto issue_step = [&]() {
    // rows written by the tile's threads -> visible to the MMA issued by thread 0 of the tile
    tmem_st_wait();
    tc_fence_before();
    asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(TPT) : "memory");
    if (lw == 0) {
      tc_fence_after();
      if (x3) {
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) tc_mma_ts(col_d, col_alo + 8 * kk, desc_hi + 16 * kk, idesc, kk > 0);
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) tc_mma_ts(col_d, col_ahi + 8 * kk, desc_lo + 16 * kk, idesc, 1);
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) tc_mma_ts(col_d, col_ahi + 8 * kk, desc_hi + 16 * kk, idesc, 1);
      } else if (blo_pass) {
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) tc_mma_ts(col_d, col_ahi + 8 * kk, desc_lo + 16 * kk, idesc, kk > 0);
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) tc_mma_ts(col_d, col_ahi + 8 * kk, desc_hi + 16 * kk, idesc, 1);
      } else {
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) tc_mma_ts(col_d, col_ahi + 8 * kk, desc_hi + 16 * kk, idesc, kk > 0);
      }
      tc_commit(my_bar);
    }
  };

  // A = identity row r of the segment (zero rows beyond the G segments); this
  // thread's column slice.
#pragma unroll
  for (int c = 0; c < NPH; c += 8) {
    if (c0 + c < KP) {
      uint32_t h[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) h[j] = (live && c0 + c + j == r) ? 0x3f800000u : 0u;
      tmem_st<8>(lane_off + col_ahi + c0 + c, h);
      if (x3) {
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = 0u;
        tmem_st<8>(lane_off + col_alo + c0 + c, h);
      }
    }
  }
  // Row value = w * 2^rexp.  The rows are rescaled (exactly, by 2^-s) only
  // when their max leaves [2^-32, 2^32]; the scale decided on one step is
  // applied on the next (warp-uniform multiply), so the common step costs one
  // multiply per column.  With H slices the row max is combined through
  // shared memory after the tile barrier that precedes the MMA issue.
  long long rexp = 0;
  int s_pend = 0;     // exponent to remove on the next step (0: none)
  float sc_fin = 1.0f;
  float last_mx = 0.0f;
  const float* e_fin = esm;
  __syncthreads();  // constants and segment table staged
  const int64_t nblk = (len_max + EB - 1) / EB;
  fill_emission_tc<NP>(args, esm, psm, sseg, 0, len_max, g_eff, rstage);
  issue_step();  // product of step 0
  __syncthreads();

  // One step of the tile.  FIRST: step 0, where the rows of a
  // one-record-shorter segment idle (keep their identity row).
  uint32_t phase = 0;
  int tstep = 0;
  auto step = [&](auto first_tag, const float* e, bool more) {
    constexpr bool FIRST = decltype(first_tag)::value;
    const bool tr = args.trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && lw == 0 && tstep < 256;
    long long t_[6];
    if (tr) t_[0] = clock64();
    mbar_wait(my_bar, phase);
    tc_fence_after();
    if (tr) t_[1] = clock64();
    uint32_t d[NPH];
    tmem_ld<NPH>(d, lane_off + col_d + c0);
    tmem_ld_wait<NPH>(d);
    if (tr) t_[2] = clock64();
    e_fin = e;
    float mx = 0.0f;
    bool active = true;
    if constexpr (FIRST) active = my_off == 0;
    const bool rescale = __any_sync(kFull, s_pend != 0);
    if (active) {
      const float4* e4 = reinterpret_cast<const float4*>(e + c0);
      if (rescale) {
        const float sc = pow2f_normal(-s_pend);
        rexp += s_pend;
        s_pend = 0;
        sc_fin = sc;
#pragma unroll
        for (int c = 0; c < NPH; c += 4) {
          const float4 ev = e4[c / 4];
          const float w0 = __uint_as_float(d[c]) * ev.x * sc, w1 = __uint_as_float(d[c + 1]) * ev.y * sc;
          const float w2 = __uint_as_float(d[c + 2]) * ev.z * sc, w3 = __uint_as_float(d[c + 3]) * ev.w * sc;
          mx = fmaxf(mx, fmaxf(fmaxf(w0, w1), fmaxf(w2, w3)));
          d[c] = __float_as_uint(w0);
          d[c + 1] = __float_as_uint(w1);
          d[c + 2] = __float_as_uint(w2);
          d[c + 3] = __float_as_uint(w3);
        }
      } else {
        sc_fin = 1.0f;
#pragma unroll
        for (int c = 0; c < NPH; c += 4) {
          const float4 ev = e4[c / 4];
          const float w0 = __uint_as_float(d[c]) * ev.x, w1 = __uint_as_float(d[c + 1]) * ev.y;
          const float w2 = __uint_as_float(d[c + 2]) * ev.z, w3 = __uint_as_float(d[c + 3]) * ev.w;
          mx = fmaxf(mx, fmaxf(fmaxf(w0, w1), fmaxf(w2, w3)));
          d[c] = __float_as_uint(w0);
          d[c + 1] = __float_as_uint(w1);
          d[c + 2] = __float_as_uint(w2);
          d[c + 3] = __float_as_uint(w3);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < NPH; ++j) d[j] = (c0 + j == r) ? 0x3f800000u : 0u;
    }
    float* slot = mxs + (static_cast<size_t>((phase & 1u) * T + wg) * H) * kTcRows;
    if (H > 1) slot[hh * kTcRows + lr] = mx;
    if (tr) t_[3] = clock64();
    if (more) {
      // Next A operand.  The tensor core reads the top 19 bits of each tf32
      // container, so adding half an ulp of tf32 rounds to nearest (ties away
      // from zero); hi is masked exactly for the 3xTF32 remainder.
#pragma unroll
      for (int c = 0; c < NPH; c += 8) {
        if (c0 + c < KP) {
          uint32_t h[8];
          if (x3) {
#pragma unroll
            for (int j = 0; j < 8; ++j) h[j] = (d[c + j] + 0x1000u) & 0xffffe000u;
            tmem_st<8>(lane_off + col_ahi + c0 + c, h);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              h[j] = __float_as_uint(__uint_as_float(d[c + j]) - __uint_as_float(h[j])) + 0x1000u;
            tmem_st<8>(lane_off + col_alo + c0 + c, h);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) h[j] = d[c + j] + 0x1000u;
            tmem_st<8>(lane_off + col_ahi + c0 + c, h);
          }
        }
      }
      if (tr) t_[4] = clock64();
      issue_step();  // includes the tile barrier: every slice's partial max is visible
      if (H > 1) {
#pragma unroll
        for (int g = 0; g < H; ++g) mx = fmaxf(mx, slot[g * kTcRows + lr]);
      }
      if (active && mx > 0.0f && (mx < 0x1p-32f || mx >= 0x1p32f)) s_pend = max(-126, min(126, ilogbf(mx)));
    }
    last_mx = mx;
    phase ^= 1u;
    if (tr) {
      t_[5] = clock64();
      if (!more) t_[4] = t_[3];
      for (int k = 0; k < 6; ++k) args.trace[(wg * 256 + tstep) * 6 + k] = t_[k];
    }
    ++tstep;
  };

  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t t0 = blk * EB;
    const int cnt = static_cast<int>(len_max - t0 < EB ? len_max - t0 : EB);
    if (blk + 1 < nblk)
      fill_emission_tc<NP>(args, esm + ((blk + 1) & 1) * esm_stride, psm, sseg, t0 + EB, len_max, g_eff, rstage);
    const float* ebuf = esm + (blk & 1) * esm_stride + static_cast<size_t>(live ? s_loc : 0) * EB * NP;
    int i = 0;
    if (blk == 0) {
      step(std::true_type{}, ebuf, 1 < len_max);
      i = 1;
    }
    for (; i < cnt; ++i) step(std::false_type{}, ebuf + i * NP, t0 + i + 1 < len_max);
    __syncthreads();
  }

  // Node (FP64 format, pitch KP = padded K): exponent E = max over the segment's
  // rows of the row-max exponent; the final rows are re-derived from the last
  // accumulator (still in TMEM) and written as w * 2^(rexp - E).
  float mx = last_mx;  // the final step's slice max; combine the slices
  if (H > 1) {
    const float* slot = mxs + (static_cast<size_t>(((phase ^ 1u) & 1u) * T + wg) * H) * kTcRows;
#pragma unroll
    for (int g = 0; g < H; ++g) mx = fmaxf(mx, slot[g * kTcRows + lr]);
  }
  if (hh == 0) rsm[row] = (live && mx > 0.0f) ? static_cast<double>(rexp + ilogbf(mx)) : -INFINITY;
  __syncthreads();
  double E = -INFINITY;
  if (live)
    for (int j = 0; j < K; ++j) E = fmax(E, rsm[s_loc * K + j]);
  tc_fence_after();
  uint32_t d[NPH];
  tmem_ld<NPH>(d, lane_off + col_d + c0);
  tmem_ld_wait<NPH>(d);
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(ncols) : "memory");
  }
  if (!live) return;
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg0 + s_loc;
  double* out = args.seg_m + node * KP * KP + static_cast<size_t>(r) * KP;
  const bool zero = (E == -INFINITY) || !(mx > 0.0f);
  const int sh = zero ? 0 : static_cast<int>(fmax(static_cast<double>(rexp) - E, -2100.0));
#pragma unroll
  for (int j = 0; j < NPH; j += 2) {
    if (c0 + j < KP) {
      double2 o;
      o.x = (zero || sh < -2044) ? 0.0
                                 : scale_pow2(static_cast<double>(__uint_as_float(d[j]) * e_fin[c0 + j] * sc_fin), sh);
      o.y = (zero || sh < -2044)
                ? 0.0
                : scale_pow2(static_cast<double>(__uint_as_float(d[j + 1]) * e_fin[c0 + j + 1] * sc_fin), sh);
      *reinterpret_cast<double2*>(out + c0 + j) = o;
    }
  }
  if (r == 0 && hh == 0) {
    for (int pr = K; pr < KP; ++pr)
      for (int c = 0; c < KP; ++c) args.seg_m[node * KP * KP + static_cast<size_t>(pr) * KP + c] = 0.0;
    args.seg_e[node] = (E == -INFINITY) ? 0.0 : E;
  }
}

}  // namespace thmm
