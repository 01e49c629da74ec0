// tf_qr_slab.cuh — register-resident slab kernels for tiled QR on sm_100a (b = 128, 256,
// 512; ib = 32 or 64).  One work item owns a 32-column slab of a tile held in FP64 DMMA
// accumulator registers (warp w: rows [w*RW, (w+1)*RW), RW = b/16), and applies whole
// inner blocks of compact-WY reflectors to it without re-reading the slab:
//
//   slab_apply   [R_s; A] <- (I - Y_s T_s^T Y_s^T) [R_s; A]  (Y_s = [I; V_s] or the explicit
//                unit-lower V_s), PAPER.md:383 / 424-427 with inner blocking (reading Z5):
//                W = R_s + V_s^T A  (per-warp-rows DMMA partials, fixed-order reduction),
//                W2 = T_s^T W (DMMA), R_s -= W2, A -= V_s W2 (DMMA into the resident slab)
//   ssrfb_reg    SSRFB item = slab_apply for s = 0..t-1
//   larfb_reg    LARFB item = slab_apply with V = V_kk copy
//   qr_slab      GEQRT / TSQRT, left-looking over 32-column slabs (PAPER.md:358-374,
//                386-406, inner blocking 637-647): apply every finished reflector group to
//                the slab, then Householder-factor the slab in shared memory with one
//                reduction (all column dots + the norm fused) and two CTA barriers per
//                column; T blocks by the column recurrence, and for ib = 64 the coupling
//                block T12 = -T11 (V1^T V2) T22 of the two 32-column halves.
//
// The arithmetic is the paper's Householder / compact-WY algorithm; only its blocking
// and summation order differ from the oracle (parity to rounding).
#pragma once
#include "tf_gemm.cuh"
#include "tf_sched.h"

namespace tf {


constexpr int SNJ = NSR / 8;            // n-blocks of a 32-column slab
constexpr int SLDW = NSR + 4;           // W / W2 row stride in smem (conflict-free B fragments)
constexpr int SLDC = 64 + 2;            // column stride of the T and R blocks in smem
constexpr int SPB = TF_WARPS * 512;     // one partial-sum buffer (16 rows of W per warp)

// [R_s; A_slab] <- Q_s^T [R_s; A_slab] for one reflector group of nw (32 or 64) columns.
//   acc : the slab (rows r0 + 8i + g, columns 8j + 2q + e), updated in place
//   Vs  : V column 0 of the group, (r, m) at Vs[r + m*b]; rows < vrow0 are zero and skipped
//   Rr  : R_s rows of the slab, (m, c) at Rr[m + c*b], or null (V has its own unit diagonal)
//   Tb  : T block of the group, (r, c) at Tb[r + c*ldt], upper triangular incl. zero lower part
template <int MI>
__device__ __forceinline__ void slab_apply(double (&acc)[MI][SNJ][2], const double* Vs, int vrow0, double* Rr,
                                           const double* Tb, int nw, int ldt, int b, double* sm) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  const bool active = r0 + RW > vrow0;  // this warp's rows meet V
  double* part = sm;                 // 2 x SPB partials (fragment order), double-buffered
  double* sW2 = sm;                  // nw x SLDW (aliases the partials after the W passes)
  double* sW = part + 2 * SPB;       // nw x SLDW
  double* sR = sW + 64 * SLDW;       // R_s, column-major, ld SLDC
  double* sT = sR + NSR * SLDC;      // T, column-major, ld SLDC
  // T and R_s land in smem by cp.async while the W passes run
  for (int x = tid; x < nw * (nw / 2); x += TF_THREADS) {
    const int c = x / (nw / 2), r = 2 * (x % (nw / 2));
    cp_async16(sT + c * SLDC + r, Tb + (size_t)c * ldt + r, 16);
  }
  if (Rr) {
    for (int x = tid; x < NSR * (nw / 2); x += TF_THREADS) {
      const int c = x / (nw / 2), r = 2 * (x % (nw / 2));
      cp_async16(sR + c * SLDC + r, Rr + r + (size_t)c * b, 16);
    }
  }
  cp_async_commit();
  TF_LU_T0();
  // B fragments (row 4*ks + q, column 8*j + g of the warp's rows) from the accumulators:
  // k-steps 2i, 2i+1 of accumulator block i in two 64-bit shuffle rounds
  const int src = 4 * q + (g >> 1);
  const bool lo = lane < 16, odd = g & 1;
  auto bpair = [&](int i, int j, double& b0, double& b1) {
    const double s1 = __shfl_sync(0xffffffffu, lo ? acc[i][j][0] : acc[i][j][1], odd ? src + 16 : src);
    const double s2 = __shfl_sync(0xffffffffu, lo ? acc[i][j][1] : acc[i][j][0], odd ? src : src + 16);
    b0 = odd ? s2 : s1;
    b1 = odd ? s1 : s2;
  };
  auto reduce = [&](int ch, const double* buf) {
    const int f = tid;  // 512 outputs, one per thread, fixed summation order
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < TF_WARPS; ++w) sum += buf[w * 512 + f];
    const int fl = f & 31, e = (f >> 5) & 1, j = (f >> 6) % SNJ, mi = (f >> 6) / SNJ;
    sW[(ch + 8 * mi + (fl >> 2)) * SLDW + 8 * j + 2 * (fl & 3) + e] = sum;
  };
  // ---- W = V^T A in passes of 16 rows (one CTA barrier per pass)
  const int np = nw / 16;
  for (int pp = 0; pp < np; ++pp) {
    const int ch = pp * 16;
    double pc[2][SNJ][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int j = 0; j < SNJ; ++j) pc[mi][j][0] = pc[mi][j][1] = 0.0;
    if (active) {
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        double a[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) a[h][mi] = Vs[(r0 + 8 * i + 4 * h + q) + (size_t)(ch + 8 * mi + g) * b];
#pragma unroll
        for (int j = 0; j < SNJ; ++j) {
          double b0, b1;
          bpair(i, j, b0, b1);
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            dmma(pc[mi][j], a[0][mi], b0);
            dmma(pc[mi][j], a[1][mi], b1);
          }
        }
#ifndef TF_SLAB_NOBOUND
        if (i & 1) asm volatile("" ::: "memory");  // bound load hoisting (register budget)
#endif
      }
    }
    double* slot = part + (pp & 1) * SPB + warp * 512;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) slot[((mi * SNJ + j) * 2 + e) * 32 + lane] = pc[mi][j][e];
    if (pp > 0) reduce(ch - 16, part + ((pp - 1) & 1) * SPB);
    if (pp == np - 1) cp_async_wait<0>();
    __syncthreads();
  }
  TF_LU_T(24);
  reduce(nw - 16, part + ((np - 1) & 1) * SPB);
  __syncthreads();
  TF_LU_T(25);
  // ---- W2 = T^T (R_s + W): T^T lower triangular -> block (mi, j) needs k < 8(mi+1)
  {
    const int bpw = nw / 32;  // 8x8 output blocks per warp (1 or 2), same mi
    const int mi = warp / (SNJ / bpw), j0 = (warp % (SNJ / bpw)) * bpw;
    double c2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int nks = 2 * (mi + 1);
    for (int ks = 0; ks < nks; ++ks) {
      const int k = 4 * ks + q;
      const double a = sT[(8 * mi + g) * SLDC + k];  // T^T(m, k) = T(k, m)
      double b0 = sW[k * SLDW + 8 * j0 + g];
      if (Rr) b0 += sR[(8 * j0 + g) * SLDC + k];
      dmma(c2[0], a, b0);
      if (bpw == 2) {
        double b1 = sW[k * SLDW + 8 * j0 + 8 + g];
        if (Rr) b1 += sR[(8 * j0 + 8 + g) * SLDC + k];
        dmma(c2[1], a, b1);
      }
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      if (x < bpw) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 8 * mi + g, c = 8 * (j0 + x) + 2 * q + e;
          sW2[m * SLDW + c] = c2[x][e];
          if (Rr) Rr[m + (size_t)c * b] = sR[c * SLDC + m] - c2[x][e];
        }
      }
    }
  }
  __syncthreads();
  TF_LU_T(26);
  // ---- A -= V W2
  if (active) {
    for (int ks = 0; ks < nw / 4; ++ks) {
      double a[MI], bq[SNJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = -Vs[(r0 + 8 * i + g) + (size_t)(4 * ks + q) * b];
#pragma unroll
      for (int j = 0; j < SNJ; ++j) bq[j] = sW2[(4 * ks + q) * SLDW + 8 * j + g];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < SNJ; ++j) dmma(acc[i][j], a[i], bq[j]);
    }
  }
  TF_LU_T(27);
  __syncthreads();  // sW2 / sT / sR / partials are rewritten by the next group
  TF_LU_T(28);
}

template <int MI>
__device__ __forceinline__ void slab_load(double (&acc)[MI][SNJ][2], const double* A, int b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * 8 * MI;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < SNJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) acc[i][j][e] = ldg_cg(A + (r0 + 8 * i + g) + (size_t)(8 * j + 2 * q + e) * b);
}

template <int MI>
__device__ __forceinline__ void slab_store(const double (&acc)[MI][SNJ][2], double* A, int b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * 8 * MI;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < SNJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) A[(r0 + 8 * i + g) + (size_t)(8 * j + 2 * q + e) * b] = acc[i][j][e];
}

// SSRFB with a shared-memory mirror of the slab (b <= 512).  The slab stays in the DMMA
// accumulators for the A update (as in slab_apply), and a copy in shared memory (rows
// swizzled so the W pass's B-fragment loads are conflict-free) feeds W = V_s^T A: the 16
// warps form two groups that each reduce over half of the rows, every warp owning whole W
// fragments over its group's rows, so W is ONE pass (per-warp K of b/2, no 16-way partial
// reduction through shared memory and no barrier per 16 W rows), the two group partials are
// added in a fixed order (group 0's + group 1's).  Then W2 = T_s^T (R_s + W) (DMMA),
// R_s -= W2, A -= V_s W2 on the accumulators, and the mirror rows are refreshed.
// Mirror layout: row r holds slab row r (32 doubles) with column c at slot (c & 7) * 4 +
// (c >> 3), so the four B-fragment values a lane of group g needs for one k-step (columns
// g, 8 + g, 16 + g, 24 + g) are adjacent (two 128-bit loads); the 16-byte chunks of a row
// are XOR-swizzled by its low two bits so the 8 lanes of each load phase (4 rows x 2 lane
// groups) hit 8 distinct bank groups.
constexpr int MIR_LD = NSR;  // mirror row length (doubles)
__device__ __forceinline__ int mir_sw(int r) { return ((r & 1) << 2) | ((r >> 1) & 1); }
__device__ __forceinline__ int mir_chunk(int r, int chunk) { return r * MIR_LD + ((chunk ^ mir_sw(r)) << 1); }

template <int MI>
__device__ inline void ssrfb_mirror(const Ctx& cx, const double* V, const double* Tst, double* R, double* A, int item,
                                    double* sm) {
  constexpr int RW = 8 * MI;
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  const int r0 = warp * RW;
  R += (size_t)item * NSR * b;
  A += (size_t)item * NSR * b;
  double* sMir = sm;                        // b x 32 (swizzled)
  double* sW = sMir + 512 * MIR_LD;         // 64 x SLDW: group-1 partials, then W, then W2
  double* sR = sW + 64 * SLDW;              // R_s, column-major, ld SLDC
  double* sT = sR + NSR * SLDC;             // T, column-major, ld SLDC
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, A, b);
  auto mirror = [&]() {
    // element (r, 8j + 2q + e): slot ((2q + e) << 2) | j, so j = 2m, 2m + 1 share chunk
    // 4q + 2e + m.  Store x of lane q writes combination (e, m) = (x + q) & 3, so the four
    // lanes of a row hit four different bank groups (with the row swizzle: all 8 lanes of
    // a store phase distinct)
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int cmb = (x + q) & 3, e = cmb >> 1, m = cmb & 1;
        const double v0 = e ? (m ? acc[i][2][1] : acc[i][0][1]) : (m ? acc[i][2][0] : acc[i][0][0]);
        const double v1 = e ? (m ? acc[i][3][1] : acc[i][1][1]) : (m ? acc[i][3][0] : acc[i][1][0]);
        *reinterpret_cast<double2*>(sMir + mir_chunk(r0 + 8 * i + g, (q << 2) | cmb)) = make_double2(v0, v1);
      }
  };
  mirror();
  const int grp = warp >> 3, wg = warp & 7;
  const int kh = b / 2, k0g = grp * kh;     // this group's rows of the W reduction
  // W tile of this warp: m-block mb, n-blocks nb0 .. nb0+NB-1 (ib = 64: 8 x 32; ib = 32: 8 x 16)
  constexpr int NBMAX = 4;
  const int NB = ib == 64 ? 4 : 2;
  const int mb = ib == 64 ? wg : (wg >> 1), nb0 = ib == 64 ? 0 : 2 * (wg & 1);
  const double* vcol0 = V + (size_t)(8 * mb + g) * b + k0g + q;  // + c0 b: V(k0g + 4ks + q, c0 + 8mb + g)
  for (int c0 = 0; c0 < b; c0 += ib) {
    const int nw = ib;
    const double* Vs = V + (size_t)c0 * b;
    const double* Tb = Tst + (size_t)c0 * ib;
    double* Rr = R + c0;
    // T_s and R_s by cp.async while W is formed
    for (int x = tid; x < nw * (nw / 2); x += TF_THREADS) {
      const int c = x / (nw / 2), r = 2 * (x % (nw / 2));
      cp_async16(sT + c * SLDC + r, Tb + (size_t)c * ib + r, 16);
    }
    for (int x = tid; x < NSR * (nw / 2); x += TF_THREADS) {
      const int c = x / (nw / 2), r = 2 * (x % (nw / 2));
      cp_async16(sR + c * SLDC + r, Rr + r + (size_t)c * b, 16);
    }
    cp_async_commit();
    __syncthreads();  // the mirror holds this block's input slab
    TF_LU_T0();
    // ---- W (nw x 32) over this group's rows: warp wg owns m-block mb, n-blocks nb0 .. nb0+NB-1
    double w[NBMAX][2];
#pragma unroll
    for (int x = 0; x < NBMAX; ++x) w[x][0] = w[x][1] = 0.0;
    const double* vcol = vcol0 + (size_t)c0 * b;
    // V operand 8 k-steps at a time, the next group in flight while this one is used
    double av[8], avn[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) avn[u] = vcol[4 * u];
    // this lane's mirror rows k0g + 4 ks + q (low bits q: a fixed swizzle), its chunks
    // (g << 1) | (n-block >> 1): addresses are the row base + immediates
    const double* mrow = sMir + (size_t)(k0g + q) * MIR_LD;
    const int sw = mir_sw(q);
    const int off0 = (((g << 1) | (nb0 >> 1)) ^ sw) << 1, off1 = (((g << 1) | 1) ^ sw) << 1;
#pragma unroll 1
    for (int ks0 = 0; ks0 < kh / 4; ks0 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) av[u] = avn[u];
      if (ks0 + 8 < kh / 4) {
#pragma unroll
        for (int u = 0; u < 8; ++u) avn[u] = vcol[4 * (ks0 + 8 + u)];
      }
      const double* rp = mrow + (size_t)ks0 * 4 * MIR_LD;
      if (NB == 4) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 lo = *reinterpret_cast<const double2*>(rp + u * 4 * MIR_LD + off0);
          const double2 hi = *reinterpret_cast<const double2*>(rp + u * 4 * MIR_LD + off1);
          dmma(w[0], av[u], lo.x);
          dmma(w[1], av[u], lo.y);
          dmma(w[2], av[u], hi.x);
          dmma(w[3], av[u], hi.y);
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 lo = *reinterpret_cast<const double2*>(rp + u * 4 * MIR_LD + off0);
          dmma(w[0], av[u], lo.x);
          dmma(w[1], av[u], lo.y);
        }
      }
    }
    TF_LU_T(24);
    // the update's first V k-step, in flight through the reduction and W2
    double an[MI];
#pragma unroll
    for (int i = 0; i < MI; ++i) an[i] = Vs[(r0 + 8 * i + g) + (size_t)q * b];
    // group 1 -> shared memory, group 0 adds (fixed order: group 0 + group 1)
    if (grp == 1) {
#pragma unroll
      for (int x = 0; x < NBMAX; ++x)
        if (x < NB)
#pragma unroll
          for (int e = 0; e < 2; ++e) sW[(8 * mb + g) * SLDW + 8 * (nb0 + x) + 2 * q + e] = w[x][e];
    }
    __syncthreads();
    if (grp == 0) {
#pragma unroll
      for (int x = 0; x < NBMAX; ++x)
        if (x < NB)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double* p = sW + (8 * mb + g) * SLDW + 8 * (nb0 + x) + 2 * q + e;
            *p = w[x][e] + *p;
          }
    }
    cp_async_wait<0>();
    __syncthreads();
    TF_LU_T(25);
    // ---- W2 = T^T (R_s + W) on the DMMA pipe (T^T lower triangular: block mi needs k < 8(mi+1))
    double c2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int bpw = nw / 32;
    const int mi = warp / (SNJ / bpw), j0 = (warp % (SNJ / bpw)) * bpw;
    {
      const int nks = 2 * (mi + 1);
      for (int ks = 0; ks < nks; ++ks) {
        const int k = 4 * ks + q;
        const double a = sT[(8 * mi + g) * SLDC + k];
        const double b0 = sW[k * SLDW + 8 * j0 + g] + sR[(8 * j0 + g) * SLDC + k];
        dmma(c2[0], a, b0);
        if (bpw == 2) {
          const double b1 = sW[k * SLDW + 8 * j0 + 8 + g] + sR[(8 * j0 + 8 + g) * SLDC + k];
          dmma(c2[1], a, b1);
        }
      }
    }
    __syncthreads();  // every warp has read W: W2 overwrites it
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      if (x < bpw) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 8 * mi + g, c = 8 * (j0 + x) + 2 * q + e;
          sW[m * SLDW + c] = c2[x][e];
          Rr[m + (size_t)c * b] = sR[c * SLDC + m] - c2[x][e];
        }
      }
    }
    __syncthreads();
    TF_LU_T(26);
    // ---- A -= V W2 on the resident accumulators (V operand one k-step ahead)
    {
      // (the sign is applied at the DMMA, where it folds into the operand modifier; negating
      // at load time costs a DADD on the FP64 pipe the DMMAs share)
      for (int ks = 0; ks < nw / 4; ++ks) {
        double a[MI], bq[SNJ];
#pragma unroll
        for (int i = 0; i < MI; ++i) a[i] = an[i];
        if (ks + 1 < nw / 4) {
#pragma unroll
          for (int i = 0; i < MI; ++i) an[i] = Vs[(r0 + 8 * i + g) + (size_t)(4 * (ks + 1) + q) * b];
        }
#pragma unroll
        for (int j = 0; j < SNJ; ++j) bq[j] = sW[(4 * ks + q) * SLDW + 8 * j + g];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < SNJ; ++j) dmma(acc[i][j], -a[i], bq[j]);
      }
    }
    TF_LU_T(27);
    // this warp's mirror rows (every warp finished reading the mirror in the W pass, which
    // precedes the W2 barriers), then the barrier before sW / sT / sR are rewritten
    if (c0 + ib < b) mirror();
    __syncthreads();
    TF_LU_T(28);
  }
  slab_store<MI>(acc, A, b);
}

// SSRFB item: 32 columns of [R_kj; A_ij] <- Q_ik^T [R_kj; A_ij], blocks s = 0..t-1.
template <int MI>
__device__ inline void ssrfb_reg(const Ctx& cx, const double* V, const double* Tst, double* R, double* A, int item,
                                 double* sm) {
  const int b = cx.b, ib = cx.ib;
  R += (size_t)item * NSR * b;
  A += (size_t)item * NSR * b;
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, A, b);
  for (int c0 = 0; c0 < b; c0 += ib) slab_apply<MI>(acc, V + (size_t)c0 * b, 0, R + c0, Tst + (size_t)c0 * ib, ib, ib, b, sm);
  slab_store<MI>(acc, A, b);
}

// LARFB item: 32 columns of A_kj <- Q_kk^T A_kj with the explicit unit-lower V_kk copy VX.
template <int MI>
__device__ inline void larfb_reg(const Ctx& cx, const double* VX, const double* Tst, double* C, int item,
                                 double* sm) {
  const int b = cx.b, ib = cx.ib;
  C += (size_t)item * NSR * b;
  double acc[MI][SNJ][2];
  slab_load<MI>(acc, C, b);
  for (int c0 = 0; c0 < b; c0 += ib)
    slab_apply<MI>(acc, VX + (size_t)c0 * b, c0, nullptr, Tst + (size_t)c0 * ib, ib, ib, b, sm);
  slab_store<MI>(acc, C, b);
}

// Householder factorization of one 32-column slab (P in smem on entry and exit: b x 32,
// column-major, ld ldp), column by column (PAPER.md:362-372 / 390-404).
//   ts   : TSQRT — reflector rows are all b rows of P, the top element of each reflector
//          is the diagonal of Rb (32 x 32, ld 33, upper part = R rows/cols of the slab),
//          whose rows receive the top components of the updates.
//   !ts  : GEQRT — column jj's reflector covers rows > cs + jj of P; row cs + jj is the top.
// Layout during the factorization: warp w keeps rows [w*RW, (w+1)*RW) (RW = b/16) and lane c
// keeps column c of them in registers.  Per column jj: every lane forms the dot of its
// column with column jj over the warp's rows (column jj's entries come from lane jj by
// shuffles), the 16 warp partials go through shared memory, and after ONE CTA barrier every
// warp sums them in the same fixed order, forms the Householder scalars itself (bitwise
// identical in all warps) and applies the rank-1 update to its rows.  Double-buffered
// partials / top rows make the single barrier per column sufficient.
template <int MI, bool TS>
__device__ inline void slab_panel(double* P, int ldp, int cs, double* Rb, double* Ts, double* sm2) {
  constexpr int RW = 8 * MI;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane, r0w = warp * RW;
  constexpr int PLD = 18;      // partials stored transposed: lane c's 16 warp partials at
                               // part[c * PLD + w] (two 128-bit loads per pair of warps,
                               // 16-byte chunks of the 8 lanes of a load phase distinct)
  double* part = sm2;          // 2 x 32 x PLD warp partials
  double* sS = part + 2 * 32 * PLD;  // 32 x 33: sdot_m of column jj (m < jj), for the T recurrence
  double* sTau = sS + 32 * 33; // 32 taus
  double* sTop = sTau + 32;    // GEQRT: 2 x 32 top rows (by column parity)
  double* Rbn = sTop + 64;     // TSQRT: 32 x 33 finished R rows (Rb stays read-only)
  double* xcol = Rbn + 32 * 33;  // 16 x RW: column jj of each warp's rows (16-byte aligned)
  double* xw = xcol + warp * RW;
  double p[RW];
#pragma unroll
  for (int k = 0; k < RW; ++k) p[k] = P[(r0w + k) + (size_t)c * ldp];
  for (int jj = 0; jj < 32; ++jj) {
    const int cg = cs + jj;
    const int kcg = cg - r0w;  // the top row's index in this warp (GEQRT)
    // warp classes (GEQRT): all rows below the top row (no masks), the warp holding the top
    // row (masks), all rows at or above it (no work); TSQRT: every row is a reflector row
    const bool full = TS || kcg < 0;
    const bool none = !TS && kcg >= RW;
    // column jj of this warp's rows, broadcast through shared memory
    __syncwarp();
    if (c == jj && !none)
#pragma unroll
      for (int k = 0; k < RW; ++k) xw[k] = p[k];
    __syncwarp();
    double d0 = 0.0, d1 = 0.0;
    if (full) {
#pragma unroll
      for (int k = 0; k < RW; k += 2) {
        const double2 x2 = *reinterpret_cast<const double2*>(xw + k);
        d0 = fma(x2.x, p[k], d0);
        d1 = fma(x2.y, p[k + 1], d1);
      }
    } else if (!none) {
#pragma unroll
      for (int k = 0; k < RW; k += 2) {
        const double2 x2 = *reinterpret_cast<const double2*>(xw + k);
        if (k > kcg) d0 = fma(x2.x, p[k], d0);
        if (k + 1 > kcg) d1 = fma(x2.y, p[k + 1], d1);
      }
    }
    double* top_row = sTop + (jj & 1) * 32;
    if (!TS && kcg >= 0 && kcg < RW) {  // publish the top row
      double tv = 0.0;
#pragma unroll
      for (int k = 0; k < RW; ++k)
        if (k == kcg) tv = p[k];
      top_row[c] = tv;
    }
    double* pb = part + (jj & 1) * 32 * PLD;
    pb[c * PLD + warp] = d0 + d1;
    __syncthreads();
    // every warp: column sums (fixed order), Householder scalars, w_c of its lane's column
    double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
    for (int w = 0; w < TF_WARPS; w += 4) {
      const double2 v01 = *reinterpret_cast<const double2*>(pb + c * PLD + w);
      const double2 v23 = *reinterpret_cast<const double2*>(pb + c * PLD + w + 2);
      e0 += v01.x;
      e1 += v01.y;
      e2 += v23.x;
      e3 += v23.y;
    }
    const double dd = (e0 + e1) + (e2 + e3);
    const double ss = __shfl_sync(0xffffffffu, dd, jj);
    const double alpha = TS ? Rb[jj * 33 + jj] : top_row[jj];
    double tau = 0.0, beta = alpha, rden = 1.0;
    if (ss != 0.0) {
      const double nrm = sqrt(alpha * alpha + ss);
      beta = (alpha >= 0.0) ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      rden = 1.0 / (alpha - beta);
    }
    const double top = TS ? (c > jj ? Rb[jj * 33 + c] : 0.0) : (c != jj ? top_row[c] : 0.0);
    const double sdot = top + dd * rden;
    const double tw = c > jj ? tau * sdot : 0.0;
    if (warp == 0) {
      if (TS && c > jj) Rbn[jj * 33 + c] = top - tw;
      if (TS && c == jj) Rbn[jj * 33 + jj] = beta;
      if (c < jj) sS[jj * 33 + c] = sdot;
      if (c == jj) sTau[jj] = tau;
    }
    // rank-1 update: p <- fac*p - tw*(x*rden); lane jj (tw = 0, fac = rden) becomes v
    const double fac = (c == jj) ? rden : 1.0;
    auto xk = [&](int k) -> double2 { return *reinterpret_cast<const double2*>(xw + k); };
    // (tw rden) x instead of tw (x rden): two FP64 operations per element instead of three
    // (the panel is bound by the FP64 pipe and its latency chain; rounding-level change)
    const double twr = tw * rden;
    if (full) {
#pragma unroll
      for (int k = 0; k < RW; k += 2) {
        const double2 x2 = xk(k);
        p[k] = fma(-twr, x2.x, p[k] * fac);
        p[k + 1] = fma(-twr, x2.y, p[k + 1] * fac);
      }
    } else if (!none) {
#pragma unroll
      for (int k = 0; k < RW; k += 2) {
        const double2 x2 = xk(k);
        if (k > kcg) p[k] = fma(-twr, x2.x, p[k] * fac);
        if (k + 1 > kcg) p[k + 1] = fma(-twr, x2.y, p[k + 1] * fac);
      }
      if (kcg >= 0) {  // GEQRT top row: R entries of row cg
#pragma unroll
        for (int k = 0; k < RW; ++k)
          if (k == kcg) p[k] = (c == jj) ? beta : p[k] - tw;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < RW; ++k) P[(r0w + k) + (size_t)c * ldp] = p[k];
  __syncthreads();
  if (TS)  // finished R rows (upper triangle incl. the diagonal)
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int rr = e / 32, cc = e % 32;
      if (rr <= cc) Rb[rr * 33 + cc] = Rbn[rr * 33 + cc];
    }
  // T (32 x 32, upper; Ts[m*33 + c] = T(m, c)) by the column recurrence, row-parallel on
  // warp 0: lane c keeps its row of T in registers (fully unrolled, static indices)
  //   T(c, jj) = -tau_jj sum_{c <= m < jj} T(c, m) sdot_jj[m],  T(c, c) = tau_c
  if (warp == 0) {
    double t[32];
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int m = 0; m < jj; ++m) {
        if (m & 1) a1 = fma(t[m], sS[jj * 33 + m], a1);
        else a0 = fma(t[m], sS[jj * 33 + m], a0);
      }
      const double tj = sTau[jj];
      t[jj] = c < jj ? -tj * (a0 + a1) : (c == jj ? tj : 0.0);
    }
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) Ts[c * 33 + jj] = t[jj];
  }
  __syncthreads();
}

// GEQRT (ts = false: A = the diagonal tile, R unused, VX = explicit unit-lower V copy)
// or TSQRT (ts = true: R = the diagonal tile's upper region, A = the tile below, VX unused),
// left-looking over 32-column slabs.  Tst: the T strip (ib x b).
template <int MI>
// Slabs [c_begin, c_end) only (multiples of 32): the slab-level DAG runs each slab as its own
// task (a slab reads only global results of the slabs before it).
__device__ inline void qr_slab(const Ctx& cx, bool ts, double* A, double* R, double* Tst, double* VX, int c_begin,
                               int c_end, double* sm) {
  const int b = cx.b, ib = cx.ib;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int RW = 8 * MI;
  const int r0 = warp * RW;
  const int ldp = b + 1;  // odd: the panel's per-lane column loads hit distinct banks
  const double* Vsrc = ts ? A : VX;
  double acc[MI][SNJ][2];
#ifdef TF_PROBE
  unsigned long long t0 = probe_now();
#endif
  for (int cs = c_begin; cs < c_end; cs += NSR) {
    const int t = cs / NSR;
    slab_load<MI>(acc, A + (size_t)cs * b, b);
    // every finished reflector group, in order
    for (int c0 = 0; c0 + ib <= cs; c0 += ib)
      slab_apply<MI>(acc, Vsrc + (size_t)c0 * b, ts ? 0 : c0, ts ? R + c0 + (size_t)cs * b : nullptr,
                     Tst + (size_t)c0 * ib, ib, ib, b, sm);
    if (ib == 64 && (t & 1))  // first half of this inner block (T11 is its T)
      slab_apply<MI>(acc, Vsrc + (size_t)(cs - 32) * b, ts ? 0 : cs - 32, ts ? R + (cs - 32) + (size_t)cs * b : nullptr,
                     Tst + (size_t)(cs - 32) * ib, 32, ib, b, sm);
    // ---- panel in shared memory
    double* P = sm;                              // b x 32, ld ldp
    double* Rb = P + 32 * ldp;                   // 32 x 33 (TSQRT)
    double* Ts = Rb + 32 * 33;                   // 32 x 33, Ts[m*33 + c] = T(m, c)
    double* sm2 = Ts + 32 * 33;                  // panel scratch (3232 + 16*RW doubles)
    double* mpart = sm2;                         // 16 x 256 (T12 products; after the panel)
    double* sM = mpart + 4096;                   // 32 x 33
    // smem: 32*ldp + 2*33*32 + 4096 + 33*32 doubles <= SMEM_USER for b <= 512
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < SNJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) P[(r0 + 8 * i + g) + (size_t)(8 * j + 2 * q + e) * ldp] = acc[i][j][e];
    if (ts)
      for (int e = tid; e < 32 * 32; e += TF_THREADS) {
        const int rr = e % 32, c = e / 32;
        Rb[rr * 33 + c] = (rr <= c) ? ldg_cg(R + (cs + rr) + (size_t)(cs + c) * b) : 0.0;
      }
    __syncthreads();
    TF_PROBE_MARK(0, t0);
    if (ts) slab_panel<MI, true>(P, ldp, cs, Rb, Ts, sm2);
    else slab_panel<MI, false>(P, ldp, cs, Rb, Ts, sm2);
    TF_PROBE_MARK(1, t0);
    // ---- results: the slab, R block (TSQRT), V copy (GEQRT), T block(s)
    {
      constexpr int CPT = 8 * MI;  // the panel's thread layout: one row, CPT columns
      const int u = lane / CPT, rw = warp * CPT + lane % CPT;
#pragma unroll 4
      for (int k = 0; k < CPT; ++k) {
        const int c = u * CPT + k;
        const double pv = P[rw + (size_t)c * ldp];
        A[rw + (size_t)(cs + c) * b] = pv;
        if (!ts) VX[rw + (size_t)(cs + c) * b] = rw > cs + c ? pv : (rw == cs + c ? 1.0 : 0.0);
      }
    }
    if (ts)
      for (int e = tid; e < 32 * 32; e += TF_THREADS) {
        const int rr = e % 32, c = e / 32;
        if (rr <= c) R[(cs + rr) + (size_t)(cs + c) * b] = Rb[rr * 33 + c];
      }
    const int s0 = (cs / ib) * ib;       // first column of this slab's inner block
    const int off = cs - s0;             // 0, or 32 for the second half of a 64-block
    for (int e = tid; e < 32 * 32; e += TF_THREADS) {
      const int rr = e % 32, c = e / 32;
      Tst[(size_t)(cs + c) * ib + off + rr] = Ts[rr * 33 + c];  // T(off + rr, off + c)
      if (ib == 64 && off == 0) Tst[(size_t)(cs + c) * ib + 32 + rr] = 0.0;  // T(32 + rr, c) = 0
    }
    if (ib == 64 && off == 32) {
      // T12 = -T11 (V1^T V2) T22; V1 = the block's first 32 columns, V2 = this slab
      const double* V1 = Vsrc + (size_t)(cs - 32) * b;
      for (int pass = 0; pass < 4; ++pass) {  // 8 rows of M = V1^T V2 per pass
        double pc[SNJ][2];
#pragma unroll
        for (int j = 0; j < SNJ; ++j) pc[j][0] = pc[j][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < RW / 4; ++ks) {
          const int rw = r0 + 4 * ks + q;
          const double a = V1[rw + (size_t)(8 * pass + g) * b];
#pragma unroll
          for (int j = 0; j < SNJ; ++j) {
            const int c = 8 * j + g;
            double bv = P[rw + (size_t)c * ldp];
            if (!ts) bv = rw > cs + c ? bv : (rw == cs + c ? 1.0 : 0.0);
            dmma(pc[j], a, bv);
          }
        }
#pragma unroll
        for (int j = 0; j < SNJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) mpart[warp * 256 + (j * 2 + e) * 32 + lane] = pc[j][e];
        __syncthreads();
        if (tid < 256) {
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < TF_WARPS; ++w) sum += mpart[w * 256 + tid];
          const int fl = tid & 31, e = (tid >> 5) & 1, j = tid >> 6;
          sM[(8 * pass + (fl >> 2)) * 33 + 8 * j + 2 * (fl & 3) + e] = sum;
        }
        __syncthreads();
      }
      // tmp = M T22 (T22 upper: k <= c), then T12 = -T11 tmp (T11 upper: m >= r)
      double tv[2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int e = tid + x * TF_THREADS, m = e % 32, c = e / 32;
        double s = 0.0;
        for (int k = 0; k <= c; ++k) s += sM[m * 33 + k] * Ts[k * 33 + c];
        tv[x] = s;
      }
      __syncthreads();
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int e = tid + x * TF_THREADS, m = e % 32, c = e / 32;
        mpart[m * 33 + c] = tv[x];
      }
      __syncthreads();
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int e = tid + x * TF_THREADS, rr = e % 32, c = e / 32;
        double s = 0.0;
        for (int m = rr; m < 32; ++m) s += ldg_cg(Tst + (size_t)(s0 + m) * ib + rr) * mpart[m * 33 + c];
        Tst[(size_t)(cs + c) * ib + rr] = -s;  // T(rr, 32 + c)
      }
    }
    __syncthreads();  // slab results (global) visible to the next slab's applies
    TF_PROBE_MARK(2, t0);
  }
}

}  // namespace tf
