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
/* (code 3 is unused: the multi-GPU data path is device-initiated peer stores over
 * CUDA IPC mappings, not NCCL; torch.distributed only exchanges the IPC handles) */
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

/* Tiled LU without pivoting — GENP, the comparison strategy of the stability study
 * (PAPER.md:865-873): Algorithm 3 with every pivot kept (GETRF keeps row j, TSTRF keeps
 * the top row), so dIpiv receives the identity encodings j+1.  Same arguments, layout and
 * info semantics as tile_lu; unstable in general (no pivoting), meant for the GETWP lab. */
int tile_lu_nopiv(int64_t n, int64_t b, int64_t ib, double* dA, double* dLs, int32_t* dIpiv,
                  int32_t* d_info, tf_stream_t stream);

/* Solves and applies with the tiled factors.
 * X: device, dense column-major n x nrhs with leading dimension ldx >= n, overwritten in
 * place (internally packed into library BDL scratch with ceil(nrhs/b) tile columns; the
 * solve runs as a DAG on the same persistent scheduler as the factorizations, reusing the
 * factorization's update kernels on the right-hand-side tiles).  dF / dT / dLs / dIpiv are
 * the (unmodified) outputs of tile_qr / tile_lu / tile_lu_nopiv with the same n, b, ib.
 * Returns 0 or -k (argument k invalid) / TF_ERR_*; no numerical checks (a zero pivot gives
 * inf / nan in X, as LAPACK getrs).  Async on `stream`.
 *   tile_getrs      X <- A^{-1} X = U^{-1} N^{-1} X   (Eq. eq:GETWPcompact, N U = A)
 *   tile_ormqr      X <- Q^T X                        (Algorithm 2's updates applied to X)
 *   tile_qrs        X <- A^{-1} X = R^{-1} Q^T X
 *   tile_lu_apply_N X <- N X  (N of Eq. eq:formula N: every elimination
 *                   step undone in reverse order; N applied to I gives N explicitly) */
int tile_getrs(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dLs, const int32_t* dIpiv,
               int64_t nrhs, double* dX, int64_t ldx, tf_stream_t stream);
int tile_ormqr(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dT, int64_t nrhs, double* dX,
               int64_t ldx, tf_stream_t stream);
int tile_qrs(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dT, int64_t nrhs, double* dX,
             int64_t ldx, tf_stream_t stream);
int tile_lu_apply_N(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dLs,
                    const int32_t* dIpiv, int64_t nrhs, double* dX, int64_t ldx, tf_stream_t stream);

/* Rectangular tiled QR / LU: Algorithm 2 / 3 on an m x n matrix of
 * p x q tiles, p = m/b, q = n/b ("p-by-q tiled matrix", 548-557), panels
 * k < min(p, q).  BDL with p tile rows: tile (i,j) at (i + j*p)*b*b.  T / L strips (i,k)
 * at (i + k*p)*ib*b and pivot vectors (i,k) at (i + k*p)*b for k < min(p, q): sizes
 * tile_mn_aux_elems / tile_mn_ipiv_elems.  Otherwise as tile_qr / tile_lu (m = n is the
 * square call). */
int tile_qr_mn(int64_t m, int64_t n, int64_t b, int64_t ib, double* dA, double* dT, tf_stream_t stream);
int tile_lu_mn(int64_t m, int64_t n, int64_t b, int64_t ib, double* dA, double* dLs, int32_t* dIpiv,
               int32_t* d_info, tf_stream_t stream);
size_t tile_mn_aux_elems(int64_t m, int64_t n, int64_t b, int64_t ib);  /* p*min(p,q)*ib*b */
size_t tile_mn_ipiv_elems(int64_t m, int64_t n, int64_t b);             /* p*min(p,q)*b */

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

/* Task-graph granularity for QR / LU on one GPU (b in {128, 256, 512}, ib in {32, 64}):
 * 1 = slab-level graph (panel tasks per 32-column slab, next-column updates per slab
 * item; the default), 0 = the paper's tile-level graph, -1 = default
 * (environment TF_FINE=0 selects tile-level).  Results are bitwise identical; applies to
 * subsequent calls on this process. */
void tile_set_slab_dag(int on);
/* Cholesky on one GPU with b a multiple of 128 (>= 256) uses the panel-level graph under
 * the same switch.  There, with min_tiles > 0, GEMM(k,i,j) outside the
 * lookahead column runs as one whole-tile work item while step k has at least `min_tiles`
 * such tiles, and as 128-row strip items afterwards; min_tiles = 0 keeps strip items
 * everywhere, -1 = default (environment TF_GEMM_TILE_MIN, else 0: measured +0.3 % speed for
 * +25 % DRAM traffic on config 4).  Results are bitwise identical; applies to
 * subsequent calls on this process. */
void tile_set_gemm_tile_min(int min_tiles);
/* Enable (cap > 0) / disable (0) the device trace: one record per work item
 * {task, item, sm, start_ns, end_ns}.  tile_trace_fetch copies the last call's records
 * (synchronizes that stream) into rec (5 int64 per record) and returns the count. */
void tile_set_trace(int64_t cap);
int64_t tile_trace_fetch(int64_t* rec, int64_t cap);
/* Grid size override for the persistent kernel (0 = one CTA per SM). */
void tile_set_ctas(int ctas);

/* Task graph export for tests / tools (host only; no device needed).  alg: 0 chol,
 * 1 qr, 2 lu; 3 getrs, 4 ormqr, 5 qrs, 6 lu_apply_N (solve DAGs with one X tile column;
 * kinds 14-22 as in tf_sched.h).  Returns the task count; fills up to `cap` entries of kind/k/i/j/level
 * (kind ids: 0 POTRF 1 TRSM 2 SYRK 3 GEMM 4 GEQRT 5 LARFB 6 TSQRT 7 SSRFB 8 GETRF
 * 9 GESSM 10 TSTRF 11 SSSSM) and the CSR successor lists (succ_off has ntasks+1
 * entries; returns edge count through *nedges).  Any output pointer may be NULL. */
int64_t tile_dag_export(int alg, int64_t p, int policy, int32_t* kind, int32_t* k, int32_t* i,
                        int32_t* j, int32_t* level, int64_t cap, int64_t* succ_off, int32_t* succ,
                        int64_t succ_cap, int64_t* nedges);

/* Slab-level task graph of QR (alg 1) / LU (alg 2) for tile size b, inner block ib (the
 * graph tile_qr / tile_lu run on one GPU when b is in {128, 256, 512} and ib in {32, 64};
 * DESIGN.md §6).  As tile_dag_export plus slab[t]: for the panel kinds 25 GEQRT-slab,
 * 26 TSQRT-slab, 27 GETRF-slab, 28 TSTRF-slab the 32-column slab the task factors; for
 * kinds 5 / 7 / 9 / 11 with one item, the slab item it runs (whole update tasks: 0).
 * Returns the task count, or -1 when (alg, b, ib) has no slab-level graph. */
int64_t tile_dag_export_slab(int alg, int64_t p, int64_t b, int64_t ib, int policy, int32_t* kind,
                             int32_t* k, int32_t* i, int32_t* j, int32_t* slab, int32_t* level,
                             int64_t cap, int64_t* succ_off, int32_t* succ, int64_t succ_cap,
                             int64_t* nedges);

/* Run one tile kernel on the given device tiles (kernel-level parity tests).
 * kind as in tile_dag_export; t0..t2 per kind:
 *   POTRF(t0=A)  TRSM(t0=L,t1=A)  SYRK(t0=A,t1=C)  GEMM(t0=A,t1=B,t2=C)
 *   GEQRT(t0=A, aux=T)  LARFB(t0=V,t1=C, aux=T)  TSQRT(t0=R,t1=A, aux=T)
 *   SSRFB(t0=V,t1=R,t2=A, aux=T)  GETRF(t0=A, ipiv)  GESSM(t0=L,t1=A, ipiv)
 *   TSTRF(t0=U,t1=A, aux=Ls, ipiv)  SSSSM(t0=L,t1=U,t2=A, aux=Ls, ipiv)
 * d_info receives the kernel's info (may be NULL). */
int tk_run(int kind, int64_t b, int64_t ib, double* t0, double* t1, double* t2, double* aux,
           int32_t* ipiv, int32_t* d_info, tf_stream_t stream);

/* ---------------------------------------------------------------------------------
 * Multi-GPU (PAPER.md:972-1049 for the DAG runtime it distributes).
 * Owner computes on a P x Q 2D block-cyclic tile grid: tile (i,j) lives on rank
 * (i mod P)*Q + (j mod Q) and every task runs on the owner of the tile it writes
 * (QR / LU: P must be 1, a column-cyclic grid, so the flat TSQRT/TSTRF chains and the
 * R/U row updates stay on one rank).  Each rank stores its tiles ("local BDL") ordered
 * column-major by local tile index: tile (i,j) at ((i/P) + (j/Q)*ceil(p/P)) * b*b; its
 * T / L strips and pivot vectors use the same local index (strip stride ib*b, pivot
 * stride b).  Panel results cross ranks inside the persistent kernel: the producing rank
 * stores the tile (L_kk / L_ik; V_kk + T_kk, V_ik + T_ik; L_kk + ipiv, L_ik + Ls + ipiv)
 * directly into each consumer's receive cache over NVLink and pushes the consumer's
 * RECV task into its ready queue with system-scope atomics; there is no host proxy.
 * Results are bitwise identical to the 1-GPU factorization (same kernels, same per-tile
 * update order).  b must be a multiple of 4; P*Q <= 8.
 *
 * Protocol (one process per GPU, all ranks collectively, in the same order):
 *   tile_dist_open    -> this rank's IPC handle (tile_dist_ipc_bytes() bytes)
 *   (gather all handles in rank order, e.g. torch.distributed.all_gather)
 *   tile_dist_connect -> maps every peer's symmetric block
 *   tile_dist_factor  -> enqueue one factorization on `stream` (repeatable)
 *   tile_dist_close
 * d_info (device int32, written at the end): LAPACK semantics combined over all ranks
 * (min failing column), or -1 if a peer did not arrive / no progress was made for
 * TF_DIST_TIMEOUT_S seconds (default 120) — a protocol timeout, never a hang.
 * Ownership: the caller owns dA_loc / dAux_loc / dIpiv_loc / d_info; the handle owns its
 * symmetric block (scheduler state + receive cache, ~p(p+1)/2 tiles when P*Q > 1). */
typedef struct tf_dist_s* tf_dist_t;

/* alg: 0 chol, 1 qr, 2 lu.  ipc_out: tile_dist_ipc_bytes() bytes (may be NULL when
 * P*Q == 1).  Returns 0 or -k / TF_ERR_* as above. */
int tile_dist_open(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, int rank, void* ipc_out,
                   tf_dist_t* out);
int tile_dist_ipc_bytes(void);
/* all_ipc: P*Q handles, rank order (this rank's own entry is ignored). */
int tile_dist_connect(tf_dist_t h, const void* all_ipc);
/* dAux_loc: T strips (qr) / L strips (lu), NULL for chol; dIpiv_loc: lu only. */
int tile_dist_factor(tf_dist_t h, double* dA_loc, double* dAux_loc, int32_t* dIpiv_loc, int32_t* d_info,
                     tf_stream_t stream);
void tile_dist_close(tf_dist_t h);
/* IPC path check (tests; no rank waits on another): tile_dist_probe enqueues on `stream`
 * one system-scope release store of `value` into peer `peer`'s probe slot for this rank
 * (through the IPC mapping made by tile_dist_connect) plus one system-scope atomic
 * increment of that peer's probe counter.  tile_dist_probe_read synchronizes the device
 * and copies this rank's own probe block to host `out`: TF_MAX_RANKS=8 slots (slot r =
 * the last value rank r stored here, 0 if none) followed by the counter (9 int32). */
int tile_dist_probe(tf_dist_t h, int peer, int32_t value, tf_stream_t stream);
int tile_dist_probe_read(tf_dist_t h, int32_t* out);
/* Elements per rank of the local buffers (same for every rank): which 0 = A (doubles),
 * 1 = T / L strips (doubles), 2 = ipiv (int32).  -1 on invalid arguments. */
int64_t tile_dist_local_elems(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, int which);
/* Owner rank of tile (i,j). */
int tile_dist_owner(int64_t i, int64_t j, int P, int Q);
/* Single-GPU emulation of a P x Q job (tests, and the only way to run the multi-rank
 * path on one GPU): ONE persistent launch whose CTAs are split into P*Q groups, each
 * running one rank's local DAG on its own local buffers (arrays of P*Q device
 * pointers); the peers' "NVLink" stores are same-device stores.  Same device code as
 * tile_dist_factor.  d_info receives the combined info. */
int tile_dist_emulate(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, double* const* dA_loc,
                      double* const* dAux_loc, int32_t* const* dIpiv_loc, int32_t* d_info,
                      tf_stream_t stream);
/* Host-only export of rank `rank`'s local task graph (tests; b = ib = 4 item counts).
 * Per local task: kind (0-11 as above, 12 SEND, 13 RECV), k, i, j (of the producing
 * task for SEND / RECV), link (SEND: offset of its entries in send_peer/send_task;
 * RECV: the producing rank; else -1), gid (global task id in program order; the
 * producer's for SEND / RECV).  CSR successors as in tile_dag_export.  send_peer /
 * send_task: the consumer rank and the RECV task id on that rank.  Returns the local
 * task count (-1 on invalid arguments). */
int64_t tile_dist_plan_export(int alg, int64_t p, int P, int Q, int rank, int32_t* kind, int32_t* k,
                              int32_t* i, int32_t* j, int32_t* link, int32_t* gid, int64_t cap,
                              int64_t* succ_off, int32_t* succ, int64_t succ_cap, int32_t* send_peer,
                              int32_t* send_task, int64_t send_cap, int64_t* nedges, int64_t* nsends);

const char* tile_strerror(int code);
const char* tile_last_error(void);
void tile_finalize(void);

#ifdef __cplusplus
}
#endif
#endif /* TILEFACT_H */
