/*
 * tilefact.h — C-ABI of libtilefact.so, the B200 (sm_100a) FP64 tiled Cholesky / QR /
 * LU library (arXiv 0709.1272; PAPER.md = the paper's text).
 *
 * Operations (each a whole factorization, executed as a dependency DAG of tile tasks
 * by one persistent device-side scheduler kernel):
 *   tile_chol — Algorithm 1 "Tiled Cholesky factorization"
 *   tile_qr   — Algorithm 2 "The tiled algorithm for QR factorization",
 *               inner blocking s = ib (§3.2.3)
 *   tile_lu   — Algorithm 3 "The tiled algorithm for LU factorization",
 *               incremental / tiled pairwise pivoting (GETWP)
 *
 * Layout — Block Data Layout: p = n/b tiles per side; tile (i,j),
 * 0-based, starts at element (i + j*p)*b*b of the matrix buffer and is column-major
 * inside (element (r,c) at r + c*b).  All values are IEEE binary64; pivots int32.
 * Factors overwrite A in place:
 *   chol: lower tiles hold L (lower triangle of diagonal tiles); upper tiles (i<j) and the
 *         strict upper triangle of diagonal tiles are never read or written.
 *   qr:   upper triangle (diagonal tiles) and tiles j>i hold R; strictly-lower part of
 *         diagonal tiles holds V_kk (unit diagonal implicit); tiles i>j hold V_ik (top
 *         part implicitly the identity).  T strips: see tile_qr_t_elems.
 *   lu:   upper triangle / tiles j>i hold U; strictly-lower part of diagonal tiles holds
 *         L_kk (unit diagonal implicit); tiles i>j hold the bottom multipliers L_ik; the
 *         top unit-lower blocks of L_ik (footnote PAPER.md:542-544) go to the L strips.
 *
 * Ownership: the caller allocates and frees every buffer it passes (device memory for
 * d* arguments).  The library owns per-(device, stream) caches of scheduler state and
 * scratch, released by tile_finalize().  Calls are asynchronous on `stream` (no host
 * synchronisation except one-time setup); calls on distinct streams with distinct
 * buffers may run concurrently.
 *
 * Return codes: 0 = enqueued; -k = argument k invalid (1-based position: n<=0, b<=0,
 * b does not divide n, ib<=0 or ib does not divide b, null pointer, b too large);
 * >0 = TF_ERR_* below.  Numerical failures are reported through d_info (device int32,
 * LAPACK semantics, written asynchronously): 0 = success; i>0 = first failing global
 * column (1-based) — chol: leading minor i not positive definite (factorization stops);
 * lu: smallest column whose pivot U(i,i) was exactly zero (factorization continues).
 * QR never fails (rank deficiency is allowed).
 */
#ifndef TILEFACT_H
#define TILEFACT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tf_stream_t; /* = cudaStream_t; NULL = legacy default stream */

#define TF_ERR_CUDA 1     /* a CUDA runtime call failed (see tile_strerror / tile_last_error) */
#define TF_ERR_NOMEM 2    /* device allocation for library scratch failed */
#define TF_ERR_NCCL 3     /* NCCL call failed (multi-GPU entry points) */
#define TF_ERR_UNSUPPORTED 4 /* configuration not supported by this build */

/* Largest tile size accepted (the in-CTA panel kernels keep O(b) state per thread). */
#define TF_MAX_B 4096

/* Tiled Cholesky, Algorithm 1.  dA: n*n doubles (BDL), in place.
 * ib: inner block for the diagonal-tile kernels (POTRF/TRSM); must divide b; it does
 * not change results beyond rounding.  d_info: 1 device int32. */
int tile_chol(int64_t n, int64_t b, int64_t ib, double* dA, int32_t* d_info, tf_stream_t stream);

/* Tiled QR, Algorithm 2.  dT: tile_qr_t_elems(n,b,ib) doubles;
 * strip (i,k), i >= k, at (i + k*p)*ib*b is ib x b column-major; inner block s occupies
 * its columns [s*ib, (s+1)*ib) and holds the upper-triangular T_s of the compact WY
 * form.  Strips with i < k are not written. */
int tile_qr(int64_t n, int64_t b, int64_t ib, double* dA, double* dT, tf_stream_t stream);

/* Tiled LU with incremental pivoting, Algorithm 3.
 * dLs: tile_lu_l_elems doubles, same strip layout as T; strip (i,k), i > k, holds the t
 * unit-lower ib x ib blocks (strictly-lower part; diagonal implicit).
 * dIpiv: tile_lu_ipiv_elems int32; vector (i,k) at (i + k*p)*b, 1-based: for (k,k) the
 * GETRF row interchanges in [1,b] (LAPACK ipiv); for (i>k,k) the TSTRF pivots in
 * [1,2b], j+1 = kept the top row, b+r+1 = bottom row r was swapped in.
 * d_info: 1 device int32. */
int tile_lu(int64_t n, int64_t b, int64_t ib, double* dA, double* dLs, int32_t* dIpiv,
            int32_t* d_info, tf_stream_t stream);

size_t tile_qr_t_elems(int64_t n, int64_t b, int64_t ib);  /* p*p*ib*b */
size_t tile_lu_l_elems(int64_t n, int64_t b, int64_t ib);  /* p*p*ib*b */
size_t tile_lu_ipiv_elems(int64_t n, int64_t b);           /* p*p*b */

/* Layout conversion: dense column-major m x n
 * (ld = m) <-> BDL tiles.  b must divide m and n.  Device pointers, async on stream. */
int tile_pack(int64_t m, int64_t n, int64_t b, const double* dDense, double* dTiles, tf_stream_t stream);
int tile_unpack(int64_t m, int64_t n, int64_t b, const double* dTiles, double* dDense, tf_stream_t stream);

/* Host-buffer convenience path (end-to-end API): copies hA (pinned or pageable host,
 * BDL) to the device, factors, copies the factors (and T / Ls / ipiv / info) back.
 * Synchronous with respect to the host on return.  Host pointers; NULL aux pointers
 * skip that copy.  kind: 0 = chol, 1 = qr, 2 = lu. */
int tile_factor_host(int kind, int64_t n, int64_t b, int64_t ib, double* hA, double* hAux,
                     int32_t* hIpiv, int32_t* hInfo, tf_stream_t stream);

/* Scheduler policy and observability (Fig. fig:flow PAPER.md:1014-1026).
 * policy: 0 = the paper's fixed kind ranks (panel > couple-factor > row-update >
 * couple-update); 1 = kind ranks plus a lookahead boost for updates of tile column k+1
 * (default).  Applies to subsequent calls on this process. */
void tile_set_policy(int policy);
/* Enable (cap > 0) / disable (0) the device trace: one record per work item
 * {task, item, sm, start_ns, end_ns}.  tile_trace_fetch copies the last call's records
 * (synchronizes that stream) into rec (5 int64 per record) and returns the count. */
void tile_set_trace(int64_t cap);
int64_t tile_trace_fetch(int64_t* rec, int64_t cap);
/* Grid size override for the persistent kernel (0 = one CTA per SM). */
void tile_set_ctas(int ctas);

/* Task graph export for tests / tools (host only; no device needed).  alg: 0 chol,
 * 1 qr, 2 lu.  Returns the task count; fills up to `cap` entries of kind/k/i/j/level
 * (kind ids: 0 POTRF 1 TRSM 2 SYRK 3 GEMM 4 GEQRT 5 LARFB 6 TSQRT 7 SSRFB 8 GETRF
 * 9 GESSM 10 TSTRF 11 SSSSM) and the CSR successor lists (succ_off has ntasks+1
 * entries; returns edge count through *nedges).  Any output pointer may be NULL. */
int64_t tile_dag_export(int alg, int64_t p, int policy, int32_t* kind, int32_t* k, int32_t* i,
                        int32_t* j, int32_t* level, int64_t cap, int64_t* succ_off, int32_t* succ,
                        int64_t succ_cap, int64_t* nedges);

/* Run one tile kernel on the given device tiles (kernel-level parity tests).
 * kind as in tile_dag_export; t0..t2 per kind:
 *   POTRF(t0=A)  TRSM(t0=L,t1=A)  SYRK(t0=A,t1=C)  GEMM(t0=A,t1=B,t2=C)
 *   GEQRT(t0=A, aux=T)  LARFB(t0=V,t1=C, aux=T)  TSQRT(t0=R,t1=A, aux=T)
 *   SSRFB(t0=V,t1=R,t2=A, aux=T)  GETRF(t0=A, ipiv)  GESSM(t0=L,t1=A, ipiv)
 *   TSTRF(t0=U,t1=A, aux=Ls, ipiv)  SSSSM(t0=L,t1=U,t2=A, aux=Ls, ipiv)
 * d_info receives the kernel's info (may be NULL). */
int tk_run(int kind, int64_t b, int64_t ib, double* t0, double* t1, double* t2, double* aux,
           int32_t* ipiv, int32_t* d_info, tf_stream_t stream);

/* Multi-GPU SPMD entry points (one call per rank, P x Q 2D block-cyclic owner-computes
 * tile distribution, tile (i,j) on rank (i mod P) + (j mod Q)*P ... see DESIGN.md §7).
 * dA_loc holds this rank's tiles ordered column-major by local (i,j); nccl_comm is an
 * ncclComm_t for the P*Q ranks.  Panel tiles are broadcast with NCCL. */
int tile_chol_dist(int64_t n, int64_t b, int64_t ib, int P, int Q, double* dA_loc,
                   int32_t* d_info, void* nccl_comm, tf_stream_t stream);
int64_t tile_dist_local_tiles(int64_t n, int64_t b, int P, int Q, int rank, int lower_only);
/* NCCL bootstrap helpers (the unique id travels over torch.distributed). */
int tile_nccl_id_bytes(void);
int tile_nccl_get_unique_id(void* id_out);
int tile_nccl_comm_init(void* id, int nranks, int rank, void** comm_out);
int tile_nccl_comm_destroy(void* comm);

const char* tile_strerror(int code);
const char* tile_last_error(void);
void tile_finalize(void);

#ifdef __cplusplus
}
#endif
#endif /* TILEFACT_H */
