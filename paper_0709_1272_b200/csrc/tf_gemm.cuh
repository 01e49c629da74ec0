// tf_gemm.cuh — CTA-wide FP64 DMMA tile-product engine (the update kernels' core).
//
// acc(BM x BN) = sum_{k<K} Aop(m,k) * Bop(k,n) for one CTA tile, with
//   Aop(m,k) at A[m + k*lda] (A_KMAJ = false, "m-contiguous") or A[k + m*lda] (true),
//   Bop(k,n) at B[n + k*ldb] (B_KMAJ = false, "n-contiguous") or B[k + n*ldb] (true).
// Rows m >= M, columns n >= N and k >= K are zero-filled, so ragged edges are exact.
// Operands stream global -> shared through an NST-stage cp.async ring of KC-deep
// slices; each warp owns a (BM/WM) x (BN/WN) sub-tile of m8n8k4 DMMA fragments held in
// registers.  The caller consumes the accumulators with for_each(f(r, c, v)).
//
// Shared layouts (doubles):  m-contig A slice: [KC][BM+4]; k-major A slice: [BM][KC+4]
// (same for B with BN).  Both paddings make the 16-lane fragment reads (4 rows x 4 k)
// hit 16 distinct bank pairs.
#pragma once
#include "tf_common.cuh"

namespace tf {

constexpr int KC = 16;    // k-depth of one pipeline slice
constexpr int NST = 3;    // pipeline stages

template <int BM, int BN, bool AK, bool BK>
struct GemmSmem {
  static constexpr int A_ELEMS = AK ? BM * (KC + 4) : KC * (BM + 4);
  static constexpr int B_ELEMS = BK ? BN * (KC + 4) : KC * (BN + 4);
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int TOTAL = NST * STAGE;  // doubles
};

template <int BM, int BN, int WM, int WN, bool AK, bool BK>
struct Gemm {
  static_assert(WM * WN == TF_WARPS, "8 warps");
  static constexpr int TM = BM / WM, TN = BN / WN;  // warp tile
  static constexpr int MI = TM / 8, NI = TN / 8;
  static_assert(MI >= 1 && NI >= 1 && TM % 8 == 0 && TN % 8 == 0, "warp tile");
  using S = GemmSmem<BM, BN, AK, BK>;
  static constexpr int SMEM_DOUBLES = S::TOTAL;

  double acc[MI][NI][2];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }

  // Issue the cp.async copies of slice `kt` into stage buffer `st`.
  template <int VEC>
  __device__ __forceinline__ static void load_slice(double* sm, int st, const double* __restrict__ A, int lda,
                                                    const double* __restrict__ B, int ldb, int M, int N, int K,
                                                    int kt) {
    double* sA = sm + st * S::STAGE;
    double* sB = sA + S::A_ELEMS;
    const int k0 = kt * KC;
    const int tid = threadIdx.x;
    // ---- A
    if (!AK) {
      constexpr int CPR = BM / VEC;  // chunks per k-row
      for (int c = tid; c < KC * CPR; c += TF_THREADS) {
        const int k = c / CPR, m = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (gk < K) ? (M - m) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (A + m + (size_t)gk * lda) : A;
        double* dst = sA + k * (BM + 4) + m;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    } else {
      constexpr int CPR = KC / VEC;
      for (int c = tid; c < BM * CPR; c += TF_THREADS) {
        const int m = c / CPR, k = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (m < M) ? (K - gk) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (A + gk + (size_t)m * lda) : A;
        double* dst = sA + m * (KC + 4) + k;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    }
    // ---- B
    if (!BK) {
      constexpr int CPR = BN / VEC;
      for (int c = tid; c < KC * CPR; c += TF_THREADS) {
        const int k = c / CPR, n = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (gk < K) ? (N - n) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (B + n + (size_t)gk * ldb) : B;
        double* dst = sB + k * (BN + 4) + n;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    } else {
      constexpr int CPR = KC / VEC;
      for (int c = tid; c < BN * CPR; c += TF_THREADS) {
        const int n = c / CPR, k = (c % CPR) * VEC;
        const int gk = k0 + k;
        int valid = (n < N) ? (K - gk) : 0;
        valid = valid < 0 ? 0 : (valid > VEC ? VEC : valid);
        const double* src = valid ? (B + gk + (size_t)n * ldb) : B;
        double* dst = sB + n * (KC + 4) + k;
        if (VEC == 2) cp_async16(dst, src, valid * 8); else cp_async8(dst, src, valid * 8);
      }
    }
  }

  __device__ __forceinline__ void compute_slice(const double* sm, int st) {
    const double* sA = sm + st * S::STAGE;
    const double* sB = sA + S::A_ELEMS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int r = lane >> 2, q = lane & 3;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int m = wm * TM + i * 8 + r;
        a[i] = AK ? sA[m * (KC + 4) + kk + q] : sA[(kk + q) * (BM + 4) + m];
      }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int n = wn * TN + j * 8 + r;
        b[j] = BK ? sB[n * (KC + 4) + kk + q] : sB[(kk + q) * (BN + 4) + n];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }

  // acc += Aop(0:M, 0:K) * Bop(0:K, 0:N).  All 256 threads must call.  On return the
  // shared buffers are free for reuse (trailing __syncthreads).
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

  __device__ __forceinline__ void run(double* sm, const double* A, int lda, const double* B, int ldb, int M,
                                      int N, int K) {
    const bool v2 = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                    ((lda | ldb) & 1) == 0;
    if (v2) run_v<2>(sm, A, lda, B, ldb, M, N, K);
    else run_v<1>(sm, A, lda, B, ldb, M, N, K);
  }

  // f(r, c, v) for every accumulator element inside [0,M) x [0,N).
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
          const int rr = wm * TM + i * 8 + r, cc = wn * TN + j * 8 + 2 * q + e;
          if (rr < M && cc < N) f(rr, cc, acc[i][j][e]);
        }
  }
};

// C(MxN, ldc) -= acc with C in global memory (L2 path).  Optional lower mask: only
// elements with (row0 + r) >= (col0 + c) are written (SYRK on a diagonal sub-tile).
template <class G>
__device__ __forceinline__ void sub_store(const G& g, double* C, int ldc, int M, int N, bool lower_mask = false,
                                          int row0 = 0, int col0 = 0) {
  g.for_each(M, N, [&](int r, int c, double v) {
    if (lower_mask && row0 + r < col0 + c) return;
    double* p = C + r + (size_t)c * ldc;
    *p = ldg_cg(p) - v;
  });
}

}  // namespace tf
