// thmm_runs.cuh -- FP64 chain kernel that absorbs runs of absent records.
//
// An absent record (no event in the hour; reference core.py:247-249) has the
// emission diagonal Q = diag(1 - p_j), the same for every absent record of a
// parameter set.  A run of r consecutive absent records therefore multiplies
// the running product by the fixed matrix
//     T_r = (Gamma Q)^r            (chain convention core.py:7-11)
// so one MMA step with T_r replaces r steps with Gamma.  Every CTA builds the
// powers T_1..T_R in its prologue (R-1 products of K x K by one warp group
// with the step machinery, ~2 us) straight into shared memory next to Gamma,
// each scaled to max in [1, 2) with its base-2 exponent; a present record is a
// step with Gamma followed by its emission scaling, exactly as in
// chain_f64_kernel.  The product is the same; only its association over an
// absent run differs (reordering-level rounding, ~1e-16 per product).
//
// Step discovery is done in the kernel from the raw present flags: one warp
// loads 32 records, ballots them, and every record that starts a step
// (present, or absent with its run position a multiple of R, runs restarting
// at each 32-record window) writes a one-byte code (0 = present, r = absent
// chunk of r records) at its prefix-popcount index.
//
// Layout: a segment's K_p rows are its own group of NT warps (rows of one
// segment share the per-step B operand, which now differs between
// segments), so groups advance independently, synchronised only by their own
// named barrier.  Nodes and exponents are written in the format of
// chain_f64_kernel, so the segment tree is shared.
#pragma once

#include "thmm_kernels.cuh"

namespace thmm {

constexpr int kRunWin = 32;  // records per discovery window (one ballot)

// Column split of the chain (as chain_f64_kernel): DMMA head tiles + SIMT
// tail states for K % 8 in 1..4 (K >= 9), else padded tiles.
__host__ __device__ constexpr int runs_split_nt(int K) {
  return (K >= 9 && K % 8 >= 1 && K % 8 <= 4) ? K / 8 : (K + 7) / 8;
}
__host__ __device__ constexpr int runs_split_tail(int K) { return (K >= 9 && K % 8 >= 1 && K % 8 <= 4) ? K % 8 : 0; }

// One table entry (Gamma or a power): head B fragments, tail couplings.
__host__ __device__ constexpr int runs_entry_pairs(int nt, int tail) {
  return nt * nt * 32 + 8 * tail * nt + (tail * tail + 1) / 2;
}
// Emission rows staged per round (present records of a window): 16, or 8
// for rows of 7+ tiles (one CTA per SM, the table takes most of the smem).
__host__ __device__ constexpr int runs_rows(int rt) { return rt >= 7 ? 8 : 16; }

// Records per discovery window: two 32-record halves, discovered by warps 0
// and 1 of the group at once (one warp when a segment has one 8-row tile).
__host__ __device__ constexpr int runs_halves(int rt) { return rt >= 2 ? 2 : 1; }

__host__ __device__ constexpr size_t runs_group_bytes(int rt) {
  return static_cast<size_t>(runs_rows(rt)) * 8 * rt * 8 +  // emission rows of up to runs_rows present records
         static_cast<size_t>(2) * kRunWin * 16 +             // staged (x, y) of the window's present records
         static_cast<size_t>(8) * rt * 8 +                   // row exponents (node epilogue)
         2 * kRunWin + 16;                                   // step codes + step / present counts per half
}

constexpr size_t kRunsSmemCap = 227 * 1024;  // opt-in shared memory per CTA (sm_100)

__host__ __device__ constexpr size_t runs_fixed_bytes(int rt) {
  return static_cast<size_t>(64) * 8 + static_cast<size_t>(8) * 8 * rt * 8;  // table exponents, constants
}

// Launch shape.  Rows of <= 4 tiles: one 32-warp CTA per SM holding a table
// of 33 entries (R = 32) when it fits, else 16-warp CTAs two per SM (<= 64
// registers either way); wider rows: one CTA per SM of 24 (5-6 tiles), 21
// (7) or 20 warps (8-10 tiles) -- whole segment groups of rt warps.
__host__ __device__ constexpr int runs_max_threads_rt(int rt) {
  return rt <= 4 ? 512 : (rt <= 6 ? 768 : (rt == 7 ? 672 : 640));
}
// groups of the one-CTA shape: 32 warps, at most 15 multi-warp groups (named
// barriers 1..15; one-warp groups synchronise with __syncwarp)
__host__ __device__ constexpr int runs_big_groups(int rt) { return rt == 1 ? 32 : (32 / rt < 15 ? 32 / rt : 15); }
// Largest R in {32, 16} whose table fits the one-CTA shape (0: neither).
__host__ __device__ constexpr int runs_big_r(int nt, int tail) {
  const size_t rest = runs_fixed_bytes(nt + (tail > 0)) +
                      static_cast<size_t>(runs_big_groups(nt + (tail > 0))) * runs_group_bytes(nt + (tail > 0));
  const size_t ent = static_cast<size_t>(runs_entry_pairs(nt, tail)) * 16;
  return 33 * ent + rest <= kRunsSmemCap ? 32 : (17 * ent + rest <= kRunsSmemCap ? 16 : 0);
}
// Table bytes one of two 16-warp CTAs per SM can hold next to its groups
// (the budget runs_r uses for that shape).
__host__ __device__ constexpr size_t runs_two_cta_budget(int rt) {
  return kRunsSmemCap / 2 - 1024 - runs_fixed_bytes(rt) -
         static_cast<size_t>(runs_max_threads_rt(rt) / (32 * rt)) * runs_group_bytes(rt);
}
// The one-CTA shape is used for rows of <= 4 tiles when it holds R = 32, or
// R = 16 where two CTAs per SM cannot fit a 17-entry table.
__host__ __device__ constexpr bool runs_big_table(int nt, int tail) {
  return nt + (tail > 0) <= 4 && runs_big_r(nt, tail) > 0 &&
         (runs_big_r(nt, tail) == 32 ||
          static_cast<size_t>(17) * runs_entry_pairs(nt, tail) * 16 > runs_two_cta_budget(nt + (tail > 0)));
}
__host__ __device__ constexpr int runs_max_threads(int nt, int tail) {
  return runs_big_table(nt, tail) ? 32 * (nt + (tail > 0)) * runs_big_groups(nt + (tail > 0))
                                  : runs_max_threads_rt(nt + (tail > 0));
}
__host__ __device__ constexpr int runs_min_blocks(int nt, int tail) {
  return (nt + (tail > 0) <= 4 && !runs_big_table(nt, tail)) ? 2 : 1;
}
// Segments (warp groups of rt warps) per CTA.
__host__ __device__ constexpr int runs_groups(int nt, int tail) {
  return runs_max_threads(nt, tail) / (32 * (nt + (tail > 0)));
}

// Longest absent chunk one step absorbs (table T_1..T_R): 32 or 16 with the
// one-CTA shape above, else the largest of 16, 8, 4, 3, 2 whose R+1 entries
// fit next to the CTA's groups.
__host__ __device__ constexpr int runs_r(int nt, int tail) {
  const int rt = nt + (tail > 0);
  const size_t budget = (runs_min_blocks(nt, tail) == 2 ? kRunsSmemCap / 2 - 1024 : kRunsSmemCap) -
                        runs_fixed_bytes(rt) - static_cast<size_t>(runs_groups(nt, tail)) * runs_group_bytes(rt);
  const size_t ent = static_cast<size_t>(runs_entry_pairs(nt, tail)) * 16;
  return runs_big_table(nt, tail)
             ? runs_big_r(nt, tail)
             : (17 * ent <= budget ? 16 : (9 * ent <= budget ? 8 : (5 * ent <= budget ? 4 : (4 * ent <= budget ? 3 : 2))));
}
__host__ __device__ constexpr int runs_r_for_k(int K) { return runs_r(runs_split_nt(K), runs_split_tail(K)); }

__host__ __device__ constexpr size_t runs_smem_bytes(int nt, int tail, int G) {
  return static_cast<size_t>(runs_r(nt, tail) + 1) * runs_entry_pairs(nt, tail) * 16 +  // table entries
         runs_fixed_bytes(nt + (tail > 0)) + static_cast<size_t>(G) * runs_group_bytes(nt + (tail > 0));
}

__device__ __forceinline__ void group_sync(int id, int threads) {
  if (threads == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
  }
}

// Emission rows of n present records (staged x, y): thread tg of the group
// evaluates state tg % KP of records tg / KP, tg / KP + GT / KP, ...  Out of
// line so the state constants never occupy the step loop's registers.
template <int KP, int GT>
__device__ __noinline__ void runs_emissions(double* ebuf, const double* psm, const double* xs, const double* ys,
                                            int n, int tg, int K) {
  const int j = tg % KP;
  const StateConsts kc = load_state_consts(psm + j, KP);
  for (int i = tg / KP; i < n; i += GT / KP) ebuf[i * KP + j] = j < K ? emission_rc(true, xs[i], ys[i], kc) : 0.0;
}

// One step's product of an 8-row tile of rows (head a, tail at) with a table
// entry: c = head-part, ct = tail columns (head DMMA tiles + SIMT coupling).
// VOLATILE_B: re-read the B fragments with ld.volatile.shared (they must not
// be hoisted out of a loop over a fixed entry -- the vector kernels' Gamma --
// into registers); the run-absorbing chain's entry changes every step, so
// plain loads there let the compiler issue them early.
template <int NT, bool SKIP, int TAIL, bool VOLATILE_B = true>
__device__ __forceinline__ void runs_mul(double (&c)[NT][2], double (&ct)[TAIL > 0 ? TAIL : 1],
                                         const double (&a)[NT][2], const double (&at)[TAIL > 0 ? TAIL : 1],
                                         const double2* ent, int lane) {
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  const int q = lane & 3;
  tile_product<NT, SKIP, VOLATILE_B>(c, a, ent, lane);
  if (TAIL > 0) {
    const double2* g21 = ent + NT * NT * 32;
    const double2* g12 = g21 + TAIL * NT * 4;
    const double* g22 = reinterpret_cast<const double*>(g12 + TAIL * NT * 4);
    // tail' = head . S12 + tail * S22 (this step's old head and tail)
#pragma unroll
    for (int j = 0; j < TAIL; ++j) {
      double sacc = 0.0;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const double2 co = lds_f64x2(g12 + (j * NT + nb) * 4 + q);
        sacc = fma(a[nb][0], co.x, sacc);
        sacc = fma(a[nb][1], co.y, sacc);
      }
      sacc += __shfl_xor_sync(kFull, sacc, 1);
      sacc += __shfl_xor_sync(kFull, sacc, 2);
#pragma unroll
      for (int i2 = 0; i2 < TAIL; ++i2) sacc = fma(at[i2], g22[i2 * TA + j], sacc);
      ct[j] = sacc;
    }
    // head' += tail (x) S21
#pragma unroll
    for (int j = 0; j < TAIL; ++j) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double2 co = lds_f64x2(g21 + (j * NT + nt) * 4 + q);
        c[nt][0] = fma(at[j], co.x, c[nt][0]);
        c[nt][1] = fma(at[j], co.y, c[nt][1]);
      }
    }
  }
}

// runs_mul in two parts, so that independent work can run between them while
// the DMMAs execute: (1) issue the head DMMAs and form tail' (from the old
// head and tail only), (2) head' += tail (x) S21 (waits for the DMMA results).
// `ent_s`: shared-window address of the entry (computed once by the caller).
template <int NT, bool SKIP, int TAIL>
__device__ __forceinline__ void runs_mul_issue(double (&c)[NT][2], double (&ct)[TAIL > 0 ? TAIL : 1],
                                               const double (&a)[NT][2], const double (&at)[TAIL > 0 ? TAIL : 1],
                                               const double2* ent, unsigned ent_s, int lane) {
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  const int q = lane & 3;
  // (tail variants keep the per-step address conversion: the precomputed base
  // measured 7 % slower at K=50 on B200, 6 % faster at K=80)
  if (TAIL == 0)
    tile_product_at<NT, SKIP>(c, a, ent_s + 16u * static_cast<unsigned>(lane));
  else
    tile_product<NT, SKIP, true>(c, a, ent, lane);
  if (TAIL > 0) {
    const unsigned g12 = ent_s + 16u * (NT * NT * 32 + TAIL * NT * 4);
    // (the tail-tail block through a plain pointer: loop-invariant, kept in registers)
    const double* g22 = reinterpret_cast<const double*>(ent + NT * NT * 32 + 2 * TAIL * NT * 4);
#pragma unroll
    for (int j = 0; j < TAIL; ++j) {
      double sacc = 0.0;
#pragma unroll
      for (int nb = 0; nb < NT; ++nb) {
        const double2 co = lds_f64x2_at(g12 + 16u * static_cast<unsigned>((j * NT + nb) * 4 + q));
        sacc = fma(a[nb][0], co.x, sacc);
        sacc = fma(a[nb][1], co.y, sacc);
      }
      sacc += __shfl_xor_sync(kFull, sacc, 1);
      sacc += __shfl_xor_sync(kFull, sacc, 2);
#pragma unroll
      for (int i2 = 0; i2 < TAIL; ++i2) sacc = fma(at[i2], g22[i2 * TA + j], sacc);
      ct[j] = sacc;
    }
  }
}
template <int NT, int TAIL>
__device__ __forceinline__ void runs_mul_couple(double (&c)[NT][2], const double (&at)[TAIL > 0 ? TAIL : 1],
                                                unsigned ent_s, int lane) {
  const int q = lane & 3;
  const unsigned g21 = ent_s + 16u * (NT * NT * 32);
#pragma unroll
  for (int j = 0; j < TAIL; ++j) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const double2 co = lds_f64x2_at(g21 + 16u * static_cast<unsigned>((j * NT + nt) * 4 + q));
      c[nt][0] = fma(at[j], co.x, c[nt][0]);
      c[nt][1] = fma(at[j], co.y, c[nt][1]);
    }
  }
}

// Stage one table entry S (element (i, j) = f(i, j), zero outside K x K) as
// head B fragments plus tail couplings.
template <int NT, int TAIL, typename F>
__device__ __forceinline__ void runs_stage_entry(double2* ent, int K, F f) {
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  for (int idx = threadIdx.x; idx < NT * NT * 32; idx += blockDim.x) {
    const int l = idx & 31, pair = idx >> 5;
    const int nb = pair % NT, nt = pair / NT;
    const int k0 = 8 * nb + 2 * (l & 3), col = 8 * nt + (l >> 2);
    const bool cin = col < K;
    ent[idx] = make_double2(cin && k0 < K ? f(k0, col) : 0.0, cin && k0 + 1 < K ? f(k0 + 1, col) : 0.0);
  }
  if (TAIL > 0) {
    double2* g21 = ent + NT * NT * 32;  // [TAIL][NT][4]: S[H+j][8nt+2q+h]
    double2* g12 = g21 + TAIL * NT * 4;  // [TAIL][NT][4]: S[8nb+2q+h][H+j]
    double* g22 = reinterpret_cast<double*>(g12 + TAIL * NT * 4);
    for (int idx = threadIdx.x; idx < TAIL * NT * 4; idx += blockDim.x) {
      const int j = idx / (NT * 4), nt = (idx >> 2) % NT, qq = idx & 3;
      const int c0 = 8 * nt + 2 * qq;
      g21[idx] = make_double2(f(H + j, c0), f(H + j, c0 + 1));
      g12[idx] = make_double2(f(c0, H + j), f(c0 + 1, H + j));
    }
    for (int idx = threadIdx.x; idx < TAIL * TAIL; idx += blockDim.x) g22[idx] = f(H + idx / TA, H + idx % TA);
  }
}

// Write the rows held by one group (the accumulator layout of the step
// loop: row 8*wg + g, head columns 8nt+2q+h, tail columns replicated in the
// quad) into a table entry's head fragments and tail couplings.
template <int NT, int TAIL>
__device__ __forceinline__ void runs_store_entry(double2* ent, const double (&c)[NT][2],
                                                 const double (&ct)[TAIL > 0 ? TAIL : 1], int row, int lane) {
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  const int q = lane & 3;
  double* e = reinterpret_cast<double*>(ent);
  if (row < H) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * nt + 2 * q + h;  // element (row, col): pair (col/8, row/8), lane (col%8, row%8/2)
        e[2 * (((col >> 3) * NT + (row >> 3)) * 32 + ((col & 7) << 2) + ((row & 7) >> 1)) + (row & 1)] = c[nt][h];
      }
    if (TAIL > 0 && q == 0) {
      double* g12 = reinterpret_cast<double*>(ent + NT * NT * 32 + TAIL * NT * 4);
#pragma unroll
      for (int j = 0; j < TAIL; ++j) g12[2 * ((j * NT + (row >> 3)) * 4 + ((row & 7) >> 1)) + (row & 1)] = ct[j];
    }
  } else if (TAIL > 0 && row < H + TAIL) {
    const int i = row - H;
    double2* g21 = ent + NT * NT * 32;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) g21[(i * NT + nt) * 4 + q] = make_double2(c[nt][0], c[nt][1]);
    if (q == 0) {
      double* g22 = reinterpret_cast<double*>(g21 + 2 * TAIL * NT * 4);
#pragma unroll
      for (int j = 0; j < TAIL; ++j) g22[i * TA + j] = ct[j];
    }
  }
}

// Load the rows of a table entry held by one group (inverse of
// runs_store_entry): head columns into the accumulator layout, tail columns
// replicated in the quad; rows >= K are zero.
template <int NT, int TAIL>
__device__ __forceinline__ void runs_load_rows(const double2* ent, double (&a)[NT][2],
                                               double (&at)[TAIL > 0 ? TAIL : 1], int row, int lane, int K) {
  constexpr int H = 8 * NT;
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  const int q = lane & 3;
  const double* e = reinterpret_cast<const double*>(ent);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) a[nt][0] = a[nt][1] = 0.0;
#pragma unroll
  for (int j = 0; j < TA; ++j) at[j] = 0.0;
  if (row >= K) return;
  if (row < H) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * nt + 2 * q + h;
        a[nt][h] = e[2 * (((col >> 3) * NT + (row >> 3)) * 32 + ((col & 7) << 2) + ((row & 7) >> 1)) + (row & 1)];
      }
    if (TAIL > 0) {
      const double* g12 = reinterpret_cast<const double*>(ent + NT * NT * 32 + TAIL * NT * 4);
#pragma unroll
      for (int j = 0; j < TAIL; ++j) at[j] = g12[2 * ((j * NT + (row >> 3)) * 4 + ((row & 7) >> 1)) + (row & 1)];
    }
  } else if (TAIL > 0) {
    const int i = row - H;
    const double2* g21 = ent + NT * NT * 32;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const double2 v = g21[(i * NT + nt) * 4 + q];
      a[nt][0] = v.x;
      a[nt][1] = v.y;
    }
    const double* g22 = reinterpret_cast<const double*>(g21 + 2 * TAIL * NT * 4);
#pragma unroll
    for (int j = 0; j < TAIL; ++j) at[j] = g22[i * TA + j];
  }
}

// ---------------------------------------------------------------------------
// Chain kernel over [lo, lo + n) in nseg equal segments (reference
// segment_bounds), G segments per CTA, RT = NT + (TAIL > 0) warps (8-row
// tiles) per segment.  Columns: NT DMMA head tiles plus TAIL SIMT tail
// states coupled by FP64 FMAs (K % 8 in 1..4, as chain_f64_kernel), else NT
// padded tiles.  Every table entry (Gamma, T_1..T_R) carries its head B
// fragments and its tail couplings.
// ---------------------------------------------------------------------------
template <int NT, bool SKIP, int TAIL>
__global__ void __launch_bounds__(runs_max_threads(NT, TAIL), runs_min_blocks(NT, TAIL))
    chain_runs_kernel(const ChainArgs args) {
  constexpr int RT = NT + (TAIL > 0 ? 1 : 0);  // 8-row tiles per segment = padded K / 8
  constexpr int KPE = 8 * RT;                    // node / emission row width
  constexpr int H = 8 * NT;                      // first tail state
  constexpr int TA = TAIL > 0 ? TAIL : 1;
  constexpr int R = runs_r(NT, TAIL);
  constexpr int MATS = R + 1;
  constexpr int ENT = runs_entry_pairs(NT, TAIL);
  constexpr int GT = RT * 32;  // threads per group
  constexpr int ROWS = runs_rows(RT);
  const int G = args.G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* tab = reinterpret_cast<double2*>(smem_raw);       // MATS entries of ENT pairs
  double* texp = reinterpret_cast<double*>(tab + MATS * ENT);  // 64
  double* psm = texp + 64;                                     // 8*KPE emission constants
  unsigned char* gbase = reinterpret_cast<unsigned char*>(psm + 8 * KPE);

  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / RT, wg = warp - grp * RT;
  const int tg = threadIdx.x - grp * GT;  // thread within the group
  const int g = lane >> 2, q = lane & 3;
  const int K = args.K;

  // ---- shared tables (whole CTA) ----
  // entry 0: Gamma; entry 1: T_1 = Gamma diag(q) scaled to max in [1, 2)
  const double* gam = args.P.gamma + static_cast<size_t>(b) * K * K;
  const double* qv = args.P.states + (static_cast<size_t>(1) * args.B + b) * K;
  runs_stage_entry<NT, TAIL>(tab, K, [&](int i, int j) { return gam[i * K + j]; });
  double m1 = 0.0;
  for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x) m1 = fmax(m1, __dmul_rn(gam[idx], qv[idx % K]));
  m1 = block_max(m1, texp, blockDim.x / 32);  // texp doubles as the reduction scratch here
  const int e1 = m1 > 0.0 ? ilogb(m1) : 0;
  auto t1 = [&](int i, int j) { return scale_pow2(__dmul_rn(gam[i * K + j], qv[j]), -e1); };
  runs_stage_entry<NT, TAIL>(tab + ENT, K, t1);
  __syncthreads();
  // entries 2..R by doubling: level k forms T_r = T_b T_{r-b} (b = 2^k) for
  // every r in (b, 2b] at once, one product per warp group (the step
  // machinery, rows of T_b loaded from its entry), each rescaled to max in
  // [1, 2) with its exponent -- ceil(log2 R) dependent products
  if (threadIdx.x == 0) {
    texp[0] = 0.0;
    texp[1] = e1;
  }
  __syncthreads();
  {
    const int row = 8 * wg + g;
    double* red = psm + grp * RT;  // per-group maxima (the emission constants are staged after this)
    for (int base = 1; base < R; base *= 2) {
      const int last = 2 * base < R ? 2 * base : R;
      for (int r0 = base + 1; r0 <= last; r0 += G) {
        const int r = r0 + grp;
        if (grp < G && r <= last) {
          double a[NT][2], at[TA], c[NT][2], ct[TA];
          runs_load_rows<NT, TAIL>(tab + base * ENT, a, at, row, lane, K);
          runs_mul<NT, SKIP, TAIL>(c, ct, a, at, tab + (r - base) * ENT, lane);
          double m = 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) m = fmax(m, fmax(c[nt][0], c[nt][1]));
#pragma unroll
          for (int j = 0; j < TAIL; ++j) m = fmax(m, ct[j]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
          if (lane == 0) red[wg] = m;
          group_sync(1 + grp, GT);
          m = red[0];
          for (int w = 1; w < RT; ++w) m = fmax(m, red[w]);
          const int ex = m > 0.0 ? ilogb(m) : 0;
          scale_row<NT>(c, ex);
#pragma unroll
          for (int j = 0; j < TAIL; ++j) ct[j] = scale_pow2(ct[j], -ex);
          runs_store_entry<NT, TAIL>(tab + r * ENT, c, ct, row, lane);
          if (wg == 0 && lane == 0) texp[r] = texp[base] + texp[r - base] + ex;
        }
        __syncthreads();
      }
    }
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
  __syncthreads();

  // ---- my segment ----
  const int64_t seg = static_cast<int64_t>(blockIdx.x) * G + grp;
  if (grp >= G || seg >= args.nseg) return;  // whole group idle (named barriers are per group)
  int64_t s_lo, s_hi;
  segment_range(args.n, args.nseg, seg, s_lo, s_hi);
  const int64_t rec0 = args.lo + s_lo, len = s_hi - s_lo;
  unsigned char* gsm = gbase + static_cast<size_t>(grp) * runs_group_bytes(RT);
  // Two halves per window from device memory; one from pinned host memory
  // (zero-copy: a second discovery warp's PCIe reads cost more than the
  // barrier cycles it saves -- measured 1.64 vs 0.65 ms per K=25 N=1e6 call).
  // (and one in collapse mode: the rank-one test runs after every 32 records)
  const int HALVES = (args.sysmem || args.collapse_tol > 0.0) ? 1 : runs_halves(RT);
  // collapse mode: windows of collapse_win (<= 32) records, the rank-one test after each
  const int WL = args.collapse_tol > 0.0 ? args.collapse_win : kRunWin;
  const int WIN = HALVES * WL;  // records per window
  double* ebuf = reinterpret_cast<double*>(gsm);  // ROWS x KPE
  double* xs = ebuf + ROWS * KPE;                 // by present rank within the window
  double* ys = xs + 2 * kRunWin;
  double* rsm = ys + 2 * kRunWin;                 // KPE row exponents
  unsigned char* code = reinterpret_cast<unsigned char*>(rsm + KPE);  // by step index within the window
  int* nstep = reinterpret_cast<int*>(code + 2 * kRunWin);  // per half: steps, present records
  const int bar = 1 + grp;

  const int row = 8 * wg + g;  // state index of my row within the segment
  const bool real = row < K;
  double a[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    a[nt][0] = (real && row == 8 * nt + 2 * q) ? 1.0 : 0.0;
    a[nt][1] = (real && row == 8 * nt + 2 * q + 1) ? 1.0 : 0.0;
  }
  double at[TA];
#pragma unroll
  for (int j = 0; j < TA; ++j) at[j] = (TAIL > 0 && real && row == H + j) ? 1.0 : 0.0;
  double rexp = 0.0;
  int since = 0;
  const int period = args.period;

  // records of the next window, prefetched into the discovery warps'
  // registers: warp h < HALVES holds record 32h + lane of the window (warp 1
  // also the present flag of record lane, to offset its half's indices)
  bool pf_valid = false, pf_pres = false, pf_valid0 = false, pf_pres0 = false;
  double pf_x = 0.0, pf_y = 0.0;
  auto prefetch = [&](int64_t wbase) {
    const int64_t t = wbase + kRunWin * wg + lane;
    pf_valid = t < len && lane < WL;
    pf_pres = false;
    pf_x = pf_y = 0.0;
    if (pf_valid) pf_pres = load_record(args, rec0 + t, pf_x, pf_y);
    if (HALVES > 1 && wg == 1) {
      pf_valid0 = wbase + lane < len;
      pf_pres0 = pf_valid0 && load_flag(args, rec0 + wbase + lane);
    }
  };
  if (wg < HALVES) prefetch(0);

  // a record starts a step: present, or absent at a run position that is a
  // multiple of R (runs restart at each 32-record half)
  auto step_starts = [&](bool valid, bool pres, unsigned P, unsigned below) {
    const unsigned pb = P & below;
    const int rstart = pb ? 32 - __clz(pb) : 0;  // one past the last present record below me
    return valid && (pres || ((lane - rstart) % R) == 0);
  };

  const int64_t nwin = (len + WIN - 1) / WIN;
  for (int64_t w = 0; w < nwin; ++w) {
    // 1. step discovery (warps 0 and 1 of the group, one 32-record half each)
    if (wg < HALVES) {
      const bool valid = pf_valid, pres = pf_pres, valid0 = pf_valid0, pres0 = pf_pres0;
      const double x = pf_x, y = pf_y;
      if (w + 1 < nwin) prefetch((w + 1) * WIN);
      const unsigned below = (1u << lane) - 1u;
      int soff = 0, poff = 0;  // steps / present records of the halves before mine
      if (HALVES > 1 && wg == 1) {
        const unsigned P0 = __ballot_sync(kFull, valid0 && pres0);
        soff = __popc(__ballot_sync(kFull, step_starts(valid0, pres0, P0, below)));
        poff = __popc(P0);
      }
      const unsigned P = __ballot_sync(kFull, valid && pres);
      const unsigned A = __ballot_sync(kFull, valid && !pres);
      const bool starts = step_starts(valid, pres, P, below);
      const unsigned S = __ballot_sync(kFull, starts);
      if (starts) {
        const int idx = soff + __popc(S & below);
        int cd = 0;
        if (pres) {
          const int pr = poff + __popc(P & below);
          xs[pr] = x;
          ys[pr] = y;
        } else {
          const unsigned rest = ~(A >> lane);
          const int run = rest ? __ffs(rest) - 1 : 32;
          cd = run < R ? run : R;
        }
        code[idx] = static_cast<unsigned char>(cd);
      }
      if (lane == 0) {
        nstep[2 * wg] = __popc(S);
        nstep[2 * wg + 1] = __popc(P);
      }
    }
    group_sync(bar, GT);
    const int ns = nstep[0] + (HALVES > 1 ? nstep[2] : 0), np = nstep[1] + (HALVES > 1 ? nstep[3] : 0);
    // 2./3. rounds of up to ROWS present records: their emission rows,
    // then the steps up to the next round's first present record
    int i = 0, prank = 0;
    for (int r0 = 0;; r0 += ROWS) {
    runs_emissions<KPE, GT>(ebuf, psm, xs + r0, ys + r0, min(np - r0, ROWS), tg, K);
    group_sync(bar, GT);
    for (; i < ns; ++i) {
      const int cd = code[i];
      if (cd == 0 && prank >= r0 + ROWS) break;  // its row comes with the next round
      double c[NT][2], ct[TA];
      runs_mul<NT, SKIP, TAIL, false>(c, ct, a, at, tab + cd * ENT, lane);
      if (cd == 0) {
        const double* erow = ebuf + (prank++ - r0) * KPE;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 ev = *reinterpret_cast<const double2*>(erow + 8 * nt + 2 * q);
          a[nt][0] = c[nt][0] * ev.x;
          a[nt][1] = c[nt][1] * ev.y;
        }
#pragma unroll
        for (int j = 0; j < TAIL; ++j) at[j] = ct[j] * erow[H + j];
      } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          a[nt][0] = c[nt][0];
          a[nt][1] = c[nt][1];
        }
#pragma unroll
        for (int j = 0; j < TAIL; ++j) at[j] = ct[j];
        rexp += texp[cd];
      }
      if (++since == period) {
        since = 0;
        renorm_row_tail<NT, TAIL>(a, at, rexp);
      }
    }
    if (i >= ns) break;
    group_sync(bar, GT);  // this round's rows consumed
    }
    group_sync(bar, GT);  // codes / rows of this window consumed
    if (args.collapse_tol > 0.0 && w + 1 < nwin) {
      // rank-one test of the product so far (thmm_vec.cuh): rows to max in
      // [1, 2); pivot p = first row with the largest exponent, j* = its
      // largest entry; row i is rho_i 2^(e_i - e_p) times the pivot when every
      // entry satisfies |m_ij - rho_i m_pj| <= tol rho_i m_pj + 2^-1022 with
      // rho_i = m_ij* / m_pj*
      renorm_row_tail<NT, TAIL>(a, at, rexp);
      since = 0;
      double rm = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) rm = fmax(rm, fmax(a[nt][0], a[nt][1]));
#pragma unroll
      for (int j = 0; j < TAIL; ++j) rm = fmax(rm, at[j]);
      rm = fmax(rm, __shfl_xor_sync(kFull, rm, 1));
      rm = fmax(rm, __shfl_xor_sync(kFull, rm, 2));
      const bool nonzero = real && rm > 0.0;
      if (q == 0) rsm[row] = nonzero ? rexp : -INFINITY;
      if (tg == 0) nstep[0] = 0;
      group_sync(bar, GT);
      int piv = -1;
      double ep = -INFINITY;
      for (int i = 0; i < K; ++i)
        if (rsm[i] > ep) {
          ep = rsm[i];
          piv = i;
        }
      double* prow = ebuf;           // the window's emission rows are consumed
      double* rho = ebuf + KPE;      // per row: rho_i
      if (row == piv) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          *reinterpret_cast<double2*>(prow + 8 * nt + 2 * q) = make_double2(a[nt][0], a[nt][1]);
        if (q == 0) {
          for (int j = H; j < KPE; ++j) prow[j] = 0.0;
#pragma unroll
          for (int j = 0; j < TAIL; ++j) prow[H + j] = at[j];
        }
      }
      group_sync(bar, GT);
      int js = 0;  // j*: first largest entry of the pivot row
      if (piv >= 0) {
        double pm = -1.0;
        for (int j = 0; j < KPE; ++j)
          if (prow[j] > pm) {
            pm = prow[j];
            js = j;
          }
      }
      // my row's entry in column j* (held by one lane of the quad, or the replicated tail)
      double vs = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        if (8 * nt + 2 * q == js) vs = a[nt][0];
        if (8 * nt + 2 * q + 1 == js) vs = a[nt][1];
      }
      vs += __shfl_xor_sync(kFull, vs, 1);
      vs += __shfl_xor_sync(kFull, vs, 2);
#pragma unroll
      for (int j = 0; j < TAIL; ++j)
        if (H + j == js) vs = at[j];
      const double rh = (piv >= 0 && nonzero) ? __ddiv_rn(vs, prow[js]) : 0.0;
      if (piv >= 0 && nonzero) {
        const double tol = args.collapse_tol, slack = 0x1p-1022;
        bool bad = !(rh > 0.0);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 pv = *reinterpret_cast<const double2*>(prow + 8 * nt + 2 * q);
          const double e0 = __dmul_rn(rh, pv.x), e1 = __dmul_rn(rh, pv.y);
          bad |= !(fabs(a[nt][0] - e0) <= fma(tol, e0, slack));
          bad |= !(fabs(a[nt][1] - e1) <= fma(tol, e1, slack));
        }
#pragma unroll
        for (int j = 0; j < TAIL; ++j) {
          const double e0 = __dmul_rn(rh, prow[H + j]);
          bad |= !(fabs(at[j] - e0) <= fma(tol, e0, slack));
        }
        if (bad) nstep[0] = 1;
      }
      if (q == 0) rho[row] = rh;
      group_sync(bar, GT);
      if (piv >= 0 && nstep[0] == 0) {
        const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg;
        for (int j = tg; j < KPE; j += GT) {
          args.col_r[node * KPE + j] = prow[j];
          const bool live = j < K && rsm[j] != -INFINITY;
          args.col_d[node * KPE + j] = live ? rsm[j] - ep : -INFINITY;
          args.col_c[node * KPE + j] = live ? rho[j] : 0.0;
        }
        if (tg == 0) {
          args.col_meta[2 * node] = static_cast<double>((w + 1) * WIN);
          args.col_meta[2 * node + 1] = ep;
        }
        return;  // the whole group leaves (named barriers are per group)
      }
      group_sync(bar, GT);  // rsm / nstep / ebuf are reused by the next window
    }
  }
  renorm_row_tail<NT, TAIL>(a, at, rexp);

  // Node exponent E = max over the segment's live rows; rows scaled to it.
  double mx = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) mx = fmax(mx, fmax(a[nt][0], a[nt][1]));
#pragma unroll
  for (int j = 0; j < TAIL; ++j) mx = fmax(mx, at[j]);
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(kFull, mx, 2));
  if (q == 0) rsm[row] = (real && mx > 0.0) ? rexp : -INFINITY;
  group_sync(bar, GT);
  double E = -INFINITY;
  for (int j = 0; j < K; ++j) E = fmax(E, rsm[j]);
  const size_t node = static_cast<size_t>(b) * args.node_stride_b + args.node_offset + seg;
  double* nrow = args.seg_m + node * KPE * KPE + static_cast<size_t>(row) * KPE;
  const bool zero = E == -INFINITY || !(mx > 0.0) || !real;
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
  if (tg == 0) {
    args.seg_e[node] = (E == -INFINITY) ? 0.0 : E;
    if (args.collapse_tol > 0.0) args.col_meta[2 * node] = -1.0;  // full node: no vector continuation
  }
}

}  // namespace thmm
