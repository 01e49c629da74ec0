// tf_gemm.cuh — CTA-wide FP64 DMMA tile-product engine (the update kernels' core).
//
// acc(BM x BN) = sum_{k<K} Aop(m,k) * Bop(k,n) for one CTA tile, with
//   Aop(m,k) at A[m + k*lda] (AK = false, "m-contiguous") or A[k + m*lda] (AK = true),
//   Bop(k,n) at B[n + k*ldb] (BK = false, "n-contiguous") or B[k + n*ldb] (BK = true).
// Rows m >= M, columns n >= N and k >= K are zero-filled, so ragged edges are exact.
// Operands stream global -> shared through an NST-stage cp.async ring of KC-deep
// slices; each of the 16 warps owns a (BM/WM) x (BN/WN) tile of m8n8k4 DMMA fragments
// in registers.  The caller consumes the accumulators with for_each(f(r, c, v)).
//
// Fragment loads are 128-bit: the MMA row / column / k labels are free (a product is
// a sum over k, and the accumulator rows/columns are relabelled in for_each), so each
// lane's two fragments are made adjacent in shared memory:
//   m-contiguous A: fragments (2i', 2i'+1) of lane row r sit at m = 16 i' + 2r + {0,1};
//   n-contiguous B: likewise over n;
//   k-major operands: k-steps are taken in pairs, lane column q reads k = 8s + 2q + {0,1}
//   (and then every operand uses that k labelling, KPERM).
// Padded strides make every 8-lane phase of a 128-bit load hit 8 distinct 16-byte bank
// groups (m/n-contiguous: stride = 4 mod 16 natural k, 2 mod 8 permuted k; k-major:
// stride KC + 8).
#pragma once
#include "tf_common.cuh"

namespace tf {

#ifdef TF_PROBE
// Phase timing probes (tools/kbench -DTF_PROBE): thread 0 accumulates globaltimer deltas.
__device__ unsigned long long* g_probe;
__device__ __forceinline__ unsigned long long probe_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TF_PROBE_MARK(slot, t0)                                                   \
  do {                                                                           \
    if (threadIdx.x == 0 && g_probe) {                                           \
      unsigned long long _t = probe_now();                                       \
      atomicAdd(&g_probe[(slot)], _t - (t0));                                    \
      t0 = _t;                                                                   \
    }                                                                            \
  } while (0)
#else
#define TF_PROBE_MARK(slot, t0) do { } while (0)
#endif

#ifndef TF_KC
#define TF_KC 32
#endif
#ifndef TF_NST
#define TF_NST 3
#endif
constexpr int KC = TF_KC;   // k-depth of one pipeline slice
constexpr int NST = TF_NST; // pipeline stages (cp.async path)
#ifndef TF_NSTB
#define TF_NSTB 6
#endif
constexpr int NSTB = TF_NSTB;  // pipeline stages of the bulk path (128x128 tiles: 6 x 33 KB)

// Dynamic shared memory per CTA and the slot reserved for the bulk pipeline's mbarriers:
// full[NSTB], empty[NSTB] and a 64-bit slice counter live in the last 16 doubles for the
// whole kernel (initialised once by pipe_init, never re-initialised).
constexpr int SMEM_DOUBLES = 25600;            // 200 KB
constexpr int PIPE_OFF = SMEM_DOUBLES - 24;    // doubles (bulk + cp.async barriers, 2 counters)
constexpr int SMEM_USER = PIPE_OFF;            // everything else fits below this

__device__ __forceinline__ uint64_t* pipe_bars(double* sm) { return reinterpret_cast<uint64_t*>(sm + PIPE_OFF); }
__device__ __forceinline__ uint64_t* pipe_bars_c(double* sm) { return pipe_bars(sm) + 2 * NSTB + 1; }

// Kernel prologue: all threads call once before any Gemm::run.
__device__ __forceinline__ void pipe_init(double* sm) {
  uint64_t* bars = pipe_bars(sm);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTB; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[NSTB + s], TF_WARPS);
    }
    bars[2 * NSTB] = 0;  // slices issued so far by this CTA (bulk path)
    uint64_t* cb = bars + 2 * NSTB + 1;  // cp.async path: full[NST] (all threads), empty[NST] (warps)
    for (int s = 0; s < NST; ++s) {
      mbar_init(&cb[s], TF_THREADS);
      mbar_init(&cb[NST + s], TF_WARPS);
    }
    cb[2 * NST] = 0;  // slices issued so far by this CTA (cp.async path)
    fence_mbar_init();
  }
  __syncthreads();
}

template <int BM, int BN, bool AK, bool BK>
struct GemmLayout {
  static constexpr bool KPERM = AK || BK;
  static constexpr int SMN_A = BM + (KPERM ? 2 : 4);  // m-contiguous A row stride (doubles)
  static constexpr int SMN_B = BN + (KPERM ? 2 : 4);
  static constexpr int SK = KC + 8;                   // k-major row stride
  static constexpr int A_ELEMS = AK ? BM * SK : KC * SMN_A;
  static constexpr int B_ELEMS = BK ? BN * SK : KC * SMN_B;
  static constexpr int STAGE = ((A_ELEMS + B_ELEMS + 1) / 2) * 2;  // keep 16-byte alignment
  static constexpr int TOTAL = NST * STAGE;                        // doubles
};

// NEG: the A fragments enter the product negated (the sign folds into the DMMA operand
// modifier), so acc += -Aop*Bop: with acc preloaded from C (load_acc) the update C -= A B
// ends with plain stores (store_acc) instead of a dependent read-modify-write epilogue.
template <int BM, int BN, int WM, int WN, bool AK, bool BK, bool NEG = false>
struct Gemm {
  static_assert(WM * WN == TF_WARPS, "all warps own a sub-tile");
  static constexpr int TM = BM / WM, TN = BN / WN;  // warp tile
  static constexpr int MI = TM / 8, NI = TN / 8;
  static_assert(TM % 16 == 0 && TN % 16 == 0, "fragments come in pairs");
  using Lay = GemmLayout<BM, BN, AK, BK>;
  static constexpr bool KPERM = Lay::KPERM;
  static constexpr int SMEM_DOUBLES = Lay::TOTAL;
  static constexpr int BM_ = BM, BN_ = BN;

  double acc[MI][NI][2];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }

  template <int VEC>
  __device__ __forceinline__ static void load_slice(double* sm, int st, const double* __restrict__ A, int lda,
                                                    const double* __restrict__ B, int ldb, int M, int N, int K,
                                                    int kt) {
    double* sA = sm + st * Lay::STAGE;
    double* sB = sA + Lay::A_ELEMS;
    const int k0 = kt * KC;
    const int tid = threadIdx.x;
    if (!AK) {
      constexpr int CPR = BM / VEC, TOT = KC * CPR;
#pragma unroll
      for (int c = tid; c < TOT; c += TF_THREADS) {
        const int k = c / CPR, m = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (gk < K) ? (M - m) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (A + m + (size_t)gk * lda) : A;
        double* dst = sA + k * Lay::SMN_A + m;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    } else {
      constexpr int CPR = KC / VEC, TOT = BM * CPR;
#pragma unroll
      for (int c = tid; c < TOT; c += TF_THREADS) {
        const int m = c / CPR, k = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (m < M) ? (K - gk) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (A + gk + (size_t)m * lda) : A;
        double* dst = sA + m * Lay::SK + k;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    }
    if (!BK) {
      constexpr int CPR = BN / VEC, TOT = KC * CPR;
#pragma unroll
      for (int c = tid; c < TOT; c += TF_THREADS) {
        const int k = c / CPR, n = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (gk < K) ? (N - n) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (B + n + (size_t)gk * ldb) : B;
        double* dst = sB + k * Lay::SMN_B + n;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    } else {
      constexpr int CPR = KC / VEC, TOT = BN * CPR;
#pragma unroll
      for (int c = tid; c < TOT; c += TF_THREADS) {
        const int n = c / CPR, k = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (n < N) ? (K - gk) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (B + gk + (size_t)n * ldb) : B;
        double* dst = sB + n * Lay::SK + k;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    }
  }

  // k row read by lane column q at k-step kk of a slice
  __device__ __forceinline__ static int kidx(int kk, int q) {
    return KPERM ? (8 * (kk >> 1) + 2 * q + (kk & 1)) : (4 * kk + q);
  }

  __device__ __forceinline__ void compute_slice(const double* sm, int st) {
    const double* sA = sm + st * Lay::STAGE;
    const double* sB = sA + Lay::A_ELEMS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
#pragma unroll
    for (int s = 0; s < KC / 8; ++s) {
      double a[2][MI], b[2][NI];  // [k-step parity][fragment]
      // ---- k-major operands: one 128-bit load covers both k-steps of the pair
      if (AK) {
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(sA + (wm * TM + 8 * i + r) * Lay::SK + 8 * s + 2 * q);
          a[0][i] = NEG ? -v.x : v.x;
          a[1][i] = NEG ? -v.y : v.y;
        }
      }
      if (BK) {
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(sB + (wn * TN + 8 * j + r) * Lay::SK + 8 * s + 2 * q);
          b[0][j] = v.x;
          b[1][j] = v.y;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = 2 * s + h;
        const int kr = kidx(kk, q);
        if (!AK) {
#pragma unroll
          for (int i2 = 0; i2 < MI / 2; ++i2) {
            const double2 v = *reinterpret_cast<const double2*>(sA + kr * Lay::SMN_A + wm * TM + 16 * i2 + 2 * r);
            a[h][2 * i2] = NEG ? -v.x : v.x;
            a[h][2 * i2 + 1] = NEG ? -v.y : v.y;
          }
        }
        if (!BK) {
#pragma unroll
          for (int j2 = 0; j2 < NI / 2; ++j2) {
            const double2 v = *reinterpret_cast<const double2*>(sB + kr * Lay::SMN_B + wn * TN + 16 * j2 + 2 * r);
            b[h][2 * j2] = v.x;
            b[h][2 * j2 + 1] = v.y;
          }
        }
#ifdef TF_M16
        if (!AK) {
          // fragment pair (2i', 2i'+1) = rows 16i' + 2r + {0,1} = one m16n8k4 (its rows r / r+8)
#pragma unroll
          for (int i2 = 0; i2 < MI / 2; ++i2)
#pragma unroll
            for (int j = 0; j < NI; ++j)
              dmma16(acc[2 * i2][j][0], acc[2 * i2][j][1], acc[2 * i2 + 1][j][0], acc[2 * i2 + 1][j][1],
                     a[h][2 * i2], a[h][2 * i2 + 1], b[h][j]);
        } else
#endif
        {
#ifdef TF_JI
#pragma unroll
          for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int i = 0; i < MI; ++i) dmma(acc[i][j], a[h][i], b[h][j]);
#else
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[h][i], b[h][j]);
#endif
        }
      }
    }
  }

  // acc += Aop(0:M, 0:K) * Bop(0:K, 0:N).  All threads must call.  On return the shared
  // buffers are free for reuse (trailing __syncthreads).
  template <int VEC>
  __device__ __forceinline__ void run_v(double* sm, const double* A, int lda, const double* B, int ldb, int M,
                                        int N, int K) {
    const int nk = (K + KC - 1) / KC;
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
      if (s < nk) load_slice<VEC>(sm, s, A, lda, B, ldb, M, N, K, s);
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<NST - 2>();
      __syncthreads();
      const int nxt = kt + NST - 1;
      if (nxt < nk) load_slice<VEC>(sm, nxt % NST, A, lda, B, ldb, M, N, K, nxt);
      cp_async_commit();
      compute_slice(sm, kt % NST);
    }
    cp_async_wait<0>();
    __syncthreads();
  }

  // cp.async ring synchronised by mbarriers instead of a CTA barrier per slice: every
  // thread issues its copies of a slice and arrives on the stage's "full" barrier when they
  // land (cp.async.mbarrier.arrive.noinc); each warp waits on "full", computes, and arrives
  // on "empty".  The refill of the stage consumed one slice earlier is issued after the
  // current slice's math, when its "empty" phase has (almost always) completed, so warps
  // drift freely inside the ring.  Stage/phase state persists across calls (slice counter).
  template <int VEC>
  __device__ __forceinline__ void run_mb(double* sm, const double* A, int lda, const double* B, int ldb, int M,
                                         int N, int K) {
    prefill_mb<VEC>(sm, A, lda, B, ldb, M, N, K);
    main_mb<VEC>(sm, A, lda, B, ldb, M, N, K);
  }

  // run_mb in two parts: prefill issues the first NST-1 slices; main_mb runs the k loop; the
  // slice counter lives in `pbase` in between.
  uint32_t pbase;
  template <int VEC>
  __device__ __forceinline__ void prefill_mb(double* sm, const double* A, int lda, const double* B, int ldb, int M,
                                             int N, int K) {
    uint64_t* full = pipe_bars_c(sm);
    uint64_t* empty = full + NST;
    uint64_t* counter = full + 2 * NST;
    const int nk = (K + KC - 1) / KC;
    pbase = (uint32_t)*reinterpret_cast<volatile uint64_t*>(counter);
    __syncthreads();  // earlier shared-memory users of the stage buffers are done
    for (int kt = 0; kt < NST - 1 && kt < nk; ++kt) {
      const uint32_t g = pbase + kt;
      const int s = g % NST;
      const uint32_t use = g / NST;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      load_slice<VEC>(sm, s, A, lda, B, ldb, M, N, K, kt);
      cp_async_mbar_arrive(&full[s]);
    }
  }
  template <int VEC>
  __device__ __forceinline__ void main_mb(double* sm, const double* A, int lda, const double* B, int ldb, int M,
                                          int N, int K) {
    uint64_t* full = pipe_bars_c(sm);
    uint64_t* empty = full + NST;
    uint64_t* counter = full + 2 * NST;
    const int nk = (K + KC - 1) / KC;
    const uint32_t base = pbase;
    auto fill = [&](int kt) {
      const uint32_t g = base + kt;
      const int s = g % NST;
      const uint32_t use = g / NST;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      load_slice<VEC>(sm, s, A, lda, B, ldb, M, N, K, kt);
      cp_async_mbar_arrive(&full[s]);
    };
    const int lane = threadIdx.x & 31;
    for (int kt = 0; kt < nk; ++kt) {
      const uint32_t g = base + kt;
      const int s = g % NST;
      mbar_wait(&full[s], (g / NST) & 1);
      compute_slice(sm, s);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (kt + NST - 1 < nk) fill(kt + NST - 1);
    }
    __syncthreads();
    *reinterpret_cast<volatile uint64_t*>(counter) = base + nk;
  }
  // nprod products sharing A, product x taking the BN operand columns at B + x * BN (Ntot
  // columns in all), run as ONE continuous slice stream through the cp.async/mbarrier ring:
  // no CTA barrier between products, and each warp hands its finished accumulators to
  // epi(x) right after its own last slice of product x, so one warp's epilogue overlaps the
  // other warps' DMMAs and the next product's slices are already in flight.  epi(x) also
  // sets up the accumulators of product x + 1 (x = -1: of product 0, called once the first
  // slices are requested): zero() or load_acc().  Same arithmetic per product as run().
  template <int VEC, class Epi>
  __device__ __forceinline__ void chain_mb(double* sm, const double* A, int lda, const double* B, int ldb, int nprod,
                                           int M, int Ntot, int K, Epi&& epi) {
    uint64_t* full = pipe_bars_c(sm);
    uint64_t* empty = full + NST;
    uint64_t* counter = full + 2 * NST;
    const int nk = (K + KC - 1) / KC;
    const int T = nk * nprod;
    const uint32_t base = (uint32_t)*reinterpret_cast<volatile uint64_t*>(counter);
    __syncthreads();  // earlier shared-memory users of the stage buffers are done
    auto fill = [&](int t) {
      const uint32_t g = base + t;
      const int s = g % NST;
      const uint32_t use = g / NST;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      const int x = t / nk, kt = t - x * nk;
      const int nn = min(BN, Ntot - x * BN);
      load_slice<VEC>(sm, s, A, lda, B + (size_t)x * BN, ldb, M, nn, K, kt);
      cp_async_mbar_arrive(&full[s]);
    };
    for (int t = 0; t < NST - 1 && t < T; ++t) fill(t);
    const int lane = threadIdx.x & 31;
    epi(-1);
    int kt = 0, x = 0;
    for (int t = 0; t < T; ++t) {
      const uint32_t g = base + t;
      const int s = g % NST;
      mbar_wait(&full[s], (g / NST) & 1);
      compute_slice(sm, s);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (t + NST - 1 < T) fill(t + NST - 1);
      if (++kt == nk) {
        epi(x);
        kt = 0;
        ++x;
      }
    }
    __syncthreads();
    *reinterpret_cast<volatile uint64_t*>(counter) = base + T;
  }
  // chain_mb over a grid of full BM x BN products: product x takes the operand rows
  // A + (x / nper) * BM and columns B + (x % nper) * BN (nper products per A strip), so a
  // whole tile's sub-tiles run as one slice stream: the pipeline fill, the last epilogue and
  // the scheduler round trip are paid once per tile instead of once per strip.  A separate
  // function (not a generalisation of chain_mb) so the strip variant keeps its registers.
  template <int VEC, class Epi>
  __device__ __forceinline__ void chain2_mb(double* sm, const double* A, int lda, const double* B, int ldb, int nprod,
                                            int nper, int K, Epi&& epi) {
    uint64_t* full = pipe_bars_c(sm);
    uint64_t* empty = full + NST;
    uint64_t* counter = full + 2 * NST;
    const int nk = (K + KC - 1) / KC;
    const int T = nk * nprod;
    const uint32_t base = (uint32_t)*reinterpret_cast<volatile uint64_t*>(counter);
    __syncthreads();  // earlier shared-memory users of the stage buffers are done
    auto fill = [&](int t) {
      const uint32_t g = base + t;
      const int s = g % NST;
      const uint32_t use = g / NST;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      const int x = t / nk, kt = t - x * nk;
      const int xa = x / nper, xb = x - xa * nper;
      load_slice<VEC>(sm, s, A + (size_t)xa * BM, lda, B + (size_t)xb * BN, ldb, BM, BN, K, kt);
      cp_async_mbar_arrive(&full[s]);
    };
    for (int t = 0; t < NST - 1 && t < T; ++t) fill(t);
    const int lane = threadIdx.x & 31;
    epi(-1);
    int kt = 0, x = 0;
    for (int t = 0; t < T; ++t) {
      const uint32_t g = base + t;
      const int s = g % NST;
      mbar_wait(&full[s], (g / NST) & 1);
      compute_slice(sm, s);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (t + NST - 1 < T) fill(t + NST - 1);
      if (++kt == nk) {
        epi(x);
        kt = 0;
        ++x;
      }
    }
    __syncthreads();
    *reinterpret_cast<volatile uint64_t*>(counter) = base + T;
  }
  template <class Epi>
  __device__ __forceinline__ void chain(double* sm, const double* A, int lda, const double* B, int ldb, int nprod,
                                        int M, int Ntot, int K, Epi&& epi) {
    if (vec2_ok(A, lda, B, ldb)) chain_mb<2>(sm, A, lda, B, ldb, nprod, M, Ntot, K, epi);
    else chain_mb<1>(sm, A, lda, B, ldb, nprod, M, Ntot, K, epi);
  }
  __device__ __forceinline__ static bool vec2_ok(const double* A, int lda, const double* B, int ldb) {
    return ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 && ((lda | ldb) & 1) == 0;
  }
  // Full-tile fast path for m/n-contiguous operands: one elected producer thread streams
  // each k-slice with bulk async copies (one per operand column, BM*8 / BN*8 bytes) into the
  // padded stage buffers and signals a per-stage "full" mbarrier by transaction bytes;
  // every warp waits on "full", computes, and arrives on the stage's "empty" mbarrier,
  // which the producer waits on before refilling.  No CTA-wide barrier per slice.
  __device__ __forceinline__ void run_bulk(double* sm, const double* A, int lda, const double* B, int ldb,
                                           int K) {
    uint64_t* full = pipe_bars(sm);
    uint64_t* empty = full + NSTB;
    uint64_t* counter = full + 2 * NSTB;
    const int nk = K / KC;
    const uint32_t base = (uint32_t)*reinterpret_cast<volatile uint64_t*>(counter);
    // Callers that stored an operand themselves issue fence_proxy_async_all() from every
    // writing thread before calling; here: all earlier shared-memory use of the stage
    // buffers is finished, and the producer orders its own view before the bulk copies.
    __syncthreads();
    if (threadIdx.x == 0) fence_proxy_async_all();
    constexpr uint32_t BYTES = (uint32_t)(KC * (BM + BN) * 8);
    // slice kt of this call is the CTA's (base + kt)-th slice: stage g % NST, use g / NST
    auto produce = [&](int kt) {
      const uint32_t g = base + kt;
      const int s = g % NSTB;
      const uint32_t use = g / NSTB;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);  // previous contents consumed
      double* sA = sm + s * Lay::STAGE;
      double* sB = sA + Lay::A_ELEMS;
      mbar_arrive_tx(&full[s], BYTES);
      const double* a = A + (size_t)kt * KC * lda;
      const double* b = B + (size_t)kt * KC * ldb;
#pragma unroll 4
      for (int k = 0; k < KC; ++k) {
        bulk_g2s(sA + k * Lay::SMN_A, a + (size_t)k * lda, BM * 8, &full[s]);
        bulk_g2s(sB + k * Lay::SMN_B, b + (size_t)k * ldb, BN * 8, &full[s]);
      }
    };
    if (threadIdx.x == 0)
      for (int kt = 0; kt < NSTB && kt < nk; ++kt) produce(kt);
    const int lane = threadIdx.x & 31;
    for (int kt = 0; kt < nk; ++kt) {
      const uint32_t g = base + kt;
      const int s = g % NSTB;
      mbar_wait(&full[s], (g / NSTB) & 1);
      compute_slice(sm, s);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (threadIdx.x == 0 && kt + NSTB < nk) produce(kt + NSTB);
    }
    __syncthreads();
    // every thread stores the same value, so each thread's next read sees base + nk
    *reinterpret_cast<volatile uint64_t*>(counter) = base + nk;
  }

  __device__ __forceinline__ void run(double* sm, const double* A, int lda, const double* B, int ldb, int M,
                                      int N, int K) {
    const bool v2 = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                    ((lda | ldb) & 1) == 0;
    // bulk pipeline only where a slice's math (BM*BN*KC/8/16 DMMAs per warp) hides the
    // producer's 2*KC copy issues: the full 128x128 tiles of GEMM / SYRK
#ifdef TF_BULK
    if (!AK && !BK && BM >= 128 && BN >= 128 && NSTB * Lay::STAGE <= SMEM_USER && v2 && M == BM && N == BN &&
        K % KC == 0 && K >= KC) {
      run_bulk(sm, A, lda, B, ldb, K);
      return;
    }
#endif
#ifdef TF_SYNC_RING
    if (v2) run_v<2>(sm, A, lda, B, ldb, M, N, K);
    else run_v<1>(sm, A, lda, B, ldb, M, N, K);
#else
    if (v2) run_mb<2>(sm, A, lda, B, ldb, M, N, K);
    else run_mb<1>(sm, A, lda, B, ldb, M, N, K);
#endif
  }

  // f(r, c, v) for every accumulator element inside [0,M) x [0,N) (undoing the labels).
  template <class F>
  __device__ __forceinline__ void for_each(int M, int N, F&& f) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int rr = AK ? (wm * TM + 8 * i + r) : (wm * TM + 16 * (i >> 1) + 2 * r + (i & 1));
          const int cl = 2 * q + e;  // local column of the C fragment = B fragment's n label
          const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
          if (rr < M && cc < N) f(rr, cc, acc[i][j][e]);
        }
  }

  // C -= acc (see sub_store).
  __device__ __forceinline__ void sub_from(double* C, int ldc, int M, int N, bool mask, int row0, int col0,
                                           bool red = false) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
    const bool vec = !AK && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((ldc & 1) == 0);
    if (!vec) {
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int rr = AK ? (wm * TM + 8 * i + r) : (wm * TM + 16 * (i >> 1) + 2 * r + (i & 1));
        double cv[NI][2];
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cl = 2 * q + e;
            const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
            cv[j][e] = (rr < M && cc < N) ? ldg_cg(C + rr + (size_t)cc * ldc) : 0.0;
          }
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cl = 2 * q + e;
            const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
            if (rr < M && cc < N && !(mask && row0 + rr < col0 + cc)) C[rr + (size_t)cc * ldc] = cv[j][e] - acc[i][j][e];
          }
      }
      return;
    }
    if (red && !AK) {
      // fire-and-forget L2 reductions: C += -acc, one IEEE add per element as C - acc (the
      // tile has a single writer at a time, so the result is the RMW's bitwise); no load
      // round trips in the epilogue
#pragma unroll
      for (int i2 = 0; i2 < MI / 2; ++i2) {
        const int rr = wm * TM + 16 * i2 + 2 * r;
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cl = 2 * q + e;
            const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
            if (cc >= N) continue;
            double* p = C + rr + (size_t)cc * ldc;
            if (rr < M && !(mask && row0 + rr < col0 + cc)) red_add_f64(p, -acc[2 * i2][j][e]);
            if (rr + 1 < M && !(mask && row0 + rr + 1 < col0 + cc)) red_add_f64(p + 1, -acc[2 * i2 + 1][j][e]);
          }
      }
      return;
    }
#pragma unroll
    for (int i2 = 0; i2 < MI / 2; ++i2) {
      const int rr = wm * TM + 16 * i2 + 2 * r;  // rows rr, rr+1 <-> acc[2*i2], acc[2*i2+1]
#pragma unroll
      for (int jb = 0; jb < NI; jb += 2) {  // batches of 4 row pairs: loads first, then stores
        double2 cv[2][2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = jb + jj, cl = 2 * q + e;
            const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
            const double* p = C + rr + (size_t)cc * ldc;
            cv[jj][e].x = cv[jj][e].y = 0.0;
            if (cc < N) {
              if (rr + 1 < M) cv[jj][e] = __ldcg(reinterpret_cast<const double2*>(p));
              else if (rr < M) cv[jj][e].x = __ldcg(p);
            }
          }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = jb + jj, cl = 2 * q + e;
            const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
            if (cc >= N) continue;
            double* p = C + rr + (size_t)cc * ldc;
            double2 v;
            v.x = cv[jj][e].x - acc[2 * i2][j][e];
            v.y = cv[jj][e].y - acc[2 * i2 + 1][j][e];
            const bool w0 = rr < M && !(mask && row0 + rr < col0 + cc);
            const bool w1 = rr + 1 < M && !(mask && row0 + rr + 1 < col0 + cc);
            if (w0 && w1) {
              *reinterpret_cast<double2*>(p) = v;
            } else {
              if (w0) p[0] = v.x;
              if (w1) p[1] = v.y;
            }
          }
      }
    }
  }

  // acc <- C (M x N block, ld ldc), the labels of sub_from; out-of-range elements 0.
  // Requires !AK (m-contiguous A: fragment rows pair up along a column of C).
  __device__ __forceinline__ void load_acc(const double* C, int ldc, int M, int N) {
    static_assert(!AK, "load_acc: m-contiguous A only");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
    const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((ldc & 1) == 0);
#pragma unroll
    for (int i2 = 0; i2 < MI / 2; ++i2) {
      const int rr = wm * TM + 16 * i2 + 2 * r;
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cl = 2 * q + e;
          const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
          const double* p = C + rr + (size_t)cc * ldc;
          double2 v = make_double2(0.0, 0.0);
          if (cc < N) {
            if (vec && rr + 1 < M) v = __ldcg(reinterpret_cast<const double2*>(p));
            else {
              if (rr < M) v.x = __ldcg(p);
              if (rr + 1 < M) v.y = __ldcg(p + 1);
            }
          }
          acc[2 * i2][j][e] = v.x;
          acc[2 * i2 + 1][j][e] = v.y;
        }
    }
  }
  // C <- acc (the labels of sub_from; optional lower mask as sub_from).
  __device__ __forceinline__ void store_acc(double* C, int ldc, int M, int N, bool mask, int row0, int col0) const {
    static_assert(!AK, "store_acc: m-contiguous A only");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
    const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((ldc & 1) == 0);
#pragma unroll
    for (int i2 = 0; i2 < MI / 2; ++i2) {
      const int rr = wm * TM + 16 * i2 + 2 * r;
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cl = 2 * q + e;
          const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
          if (cc >= N) continue;
          double* p = C + rr + (size_t)cc * ldc;
          const bool w0 = rr < M && !(mask && row0 + rr < col0 + cc);
          const bool w1 = rr + 1 < M && !(mask && row0 + rr + 1 < col0 + cc);
          if (w0 && w1 && vec) {
            *reinterpret_cast<double2*>(p) = make_double2(acc[2 * i2][j][e], acc[2 * i2 + 1][j][e]);
          } else {
            if (w0) p[0] = acc[2 * i2][j][e];
            if (w1) p[1] = acc[2 * i2 + 1][j][e];
          }
        }
    }
  }

  // f(j, e, row, col) over the in-range elements of accumulator row-fragment i.
  template <class F>
  __device__ __forceinline__ void for_row(int i, int M, int N, F&& f) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
    const int rr = AK ? (wm * TM + 8 * i + r) : (wm * TM + 16 * (i >> 1) + 2 * r + (i & 1));
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cl = 2 * q + e;
        const int cc = BK ? (wn * TN + 8 * j + cl) : (wn * TN + 16 * (j >> 1) + 2 * cl + (j & 1));
        if (rr < M && cc < N) f(j, e, rr, cc);
      }
  }
};

// C(MxN, ldc) -= acc with C in global memory (L2 path).  Optional lower mask: only
// elements with (row0 + r) >= (col0 + c) are written (SYRK on a diagonal sub-tile).
// For m-contiguous A the two rows of a fragment pair are adjacent in a column of C, so
// the read-modify-write uses 128-bit accesses, with all loads of a row pair issued
// before any store (one L2 round trip per pair instead of one per element).
// red: subtract with L2 reductions (red.global.add.f64) instead of load + store — for task
// epilogues whose C is not read back by the same CTA within the item (GEMM / SYRK).
template <class G>
__device__ __forceinline__ void sub_store(const G& g, double* C, int ldc, int M, int N, bool lower_mask = false,
                                          int row0 = 0, int col0 = 0, bool red = false) {
  g.sub_from(C, ldc, M, N, lower_mask, row0, col0, red);
}

// Warm L2 with the M x N block of C (column-major, ld ldc) ahead of its epilogue.
__device__ __forceinline__ void prefetch_l2(const double* C, int ldc, int M, int N) {
  const int lpc = (M * 8 + 127) / 128;  // 128-byte lines per column
  for (int e = threadIdx.x; e < lpc * N; e += TF_THREADS) {
    const double* p = C + (size_t)(e / lpc) * ldc + (e % lpc) * 16;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

}  // namespace tf
