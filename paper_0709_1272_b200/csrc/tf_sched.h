// tf_sched.h — data structures shared by the device scheduler (tf_device.cu) and the
// host side (tf_host.cpp): task descriptors, per-factorization problem/scheduler state,
// the multi-GPU rank context, and the launch wrappers the host calls.
//
// Execution model: the DAG of Algorithms 1-3 runs inside ONE
// persistent kernel; a task is split into work items (sub-tiles / row blocks / column
// slabs) that the CTAs pop from global-memory priority queues.  Multi-GPU:
// each rank runs the same kernel over the tasks it owns (owner computes on a P x Q
// block-cyclic tile grid); panel tiles cross ranks as SEND work items that store the
// tile straight into the consumer rank's receive cache over NVLink (peer pointers) and
// then push the consumer's RECV task into its ready queue with remote atomics.
#pragma once
#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define TF_HD __host__ __device__
#else
#define TF_HD
#endif

namespace tf {

constexpr int NLEV = 4;              // priority levels
constexpr int RB = 128;              // TRSM row block / SYRK-GEMM sub-tile edge
constexpr int NS = 64;               // column-slab width of LARFB/SSRFB/GESSM/SSSSM items
constexpr int TF_MAX_RANKS = 8;      // ranks per persistent launch (emulation) / per job
constexpr int SEND_CHUNKS = 8;       // work items per (SEND task, peer)

// task kinds: 0 POTRF 1 TRSM 2 SYRK 3 GEMM 4 GEQRT 5 LARFB 6 TSQRT 7 SSRFB
//             8 GETRF 9 GESSM 10 TSTRF 11 SSSSM 12 SEND 13 RECV
// solve / apply tasks on right-hand-side tiles X(i,c) (tf_solve.cuh; j = c):
//             14 UNITL(k) 15 XGESSM(k,c) 16 XSSSSM(i,k,c) 17 XLARFB(k,c) 18 XSSRFB(i,k,c)
//             19 XTRSMU(k,c) 20 XGEMM(i,k,c) 21 XUNSSSSM(i,k,c) 22 XUNGESSM(k,c)
constexpr int K_SEND = 12, K_RECV = 13;
constexpr int K_UNITL = 14, K_XGESSM = 15, K_XSSSSM = 16, K_XLARFB = 17, K_XSSRFB = 18, K_XTRSMU = 19,
              K_XGEMM = 20, K_XUNSSSSM = 21, K_XUNGESSM = 22;
// DAG algorithms: 0 chol, 1 qr, 2 lu (factorizations); 3 getrs (X <- A^{-1} X with LU
// factors), 4 ormqr (X <- Q^T X), 5 qrs (X <- R^{-1} Q^T X), 6 lu_apply_N (X <- N X)
constexpr int ALG_GETRS = 3, ALG_ORMQR = 4, ALG_QRS = 5, ALG_LUN = 6;
// host <-> device overlap (tile_factor_host): ARRIVE(j) is completed by the scheduler when
// tile column j has been copied in (a flag written by the copy stream); DONE(j) runs when
// every tile of column j is final and sets the flag the D2H copy stream waits on
constexpr int K_ARRIVE = 23, K_DONE = 24;
// slab-level DAG (QR / LU on the register-slab path, single GPU): the panel tasks of
// Algorithms 2-3 run as one task per 32-column slab (pad = slab), and the update tasks of
// the next panel column (j = k + 1) as one task per slab item (pad = item offset), so that
// consecutive TSQRT / TSTRF of a column and the next panel pipeline slab by slab
// (DESIGN.md §6); the arithmetic of every tile is unchanged.
// K_TSQRT_A / K_TSTRF_A: the older inner blocks of a TSQRT / TSTRF slab (pad = slab),
// applied off the critical path; the slab task then applies only the newest one and
// factors the slab.
constexpr int K_GEQRT_S = 25, K_TSQRT_S = 26, K_GETRF_S = 27, K_TSTRF_S = 28, K_TSQRT_A = 29, K_TSTRF_A = 30;
// Measured: the split shortens config 3 (LU, 10.2 -> 9.8 ms) but lengthens config 2 (QR,
// 13.0 -> 14.2 ms: the QR slab's panel dominates and the extra hop costs more than the
// applies it removes from the chain), so only TSTRF is split.
TF_HD inline bool ts_apply_split(bool lu) { return lu; }
// panel-level DAG (Cholesky, b a multiple of 128, >= 256, single GPU): POTRF(k) runs as one
// task per 128-column panel J (pad = J / 128) for the diagonal block (K_POTRF_D: update from
// the panels to its left, then the 128 x 128 factorization) and one for the blocks below it
// (K_POTRF_B: one item per 128-row block, update then triangular solve); TRSM(k,i) as one
// task per panel (K_TRSM_P, one item per 128-row block), so the TRSMs of a column start
// after the first diagonal block instead of after the whole POTRF.
constexpr int K_POTRF_D = 31, K_POTRF_B = 32, K_TRSM_P = 33;
TF_HD inline bool chol_panel_ok(int b) { return b >= 256 && b % 128 == 0; }
TF_HD inline int coarse_kind(int kind) {
  if (kind == K_POTRF_D || kind == K_POTRF_B) return 0;
  if (kind == K_TRSM_P) return 1;
  return kind == K_GEQRT_S ? 4 : (kind == K_TSQRT_S || kind == K_TSQRT_A) ? 6 : kind == K_GETRF_S ? 8
       : (kind == K_TSTRF_S || kind == K_TSTRF_A) ? 10 : kind;
}

TF_HD inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Register-slab kernels (tf_qr_slab.cuh: SSRFB / LARFB items of NSR columns, slab-wise
// GEQRT / TSQRT; tf_lu_slab.cuh: GESSM / SSSSM items): b in {128, 256, 512}, ib in {32, 64}.
constexpr int NSR = 32;
// (exactly the tile sizes TF_SLAB_DISPATCH instantiates: MI = b/128 in {1, 2, 4})
TF_HD inline bool ssrfb_reg_ok(int b, int ib) { return (b == 128 || b == 256 || b == 512) && (ib == 32 || ib == 64); }

// GEMM items cover gemm_group(b) adjacent 128x128 sub-tiles of one row strip (TF_GEMM_GROUP
// caps it; 1 = one sub-tile per item)
#ifndef TF_GEMM_GROUP
#define TF_GEMM_GROUP 4
#endif
TF_HD inline int gemm_group(int b) {
  const int nr = ceil_div(b, RB);
  int gsz = 1;
  while (gsz * 2 <= TF_GEMM_GROUP && nr % (gsz * 2) == 0) gsz *= 2;
  return gsz;
}

TF_HD inline int items_of(int kind, int b, int ib) {
  const int nr = ceil_div(b, RB);
  switch (kind) {
    case 1: return nr;                 // TRSM: row blocks
    case 2: return nr * (nr + 1) / 2;  // SYRK: lower sub-tiles
    case 3: return nr * nr / gemm_group(b);  // GEMM: groups of sub-tiles
    case 5: case 7: case 9: case 11:
    case K_XGESSM: case K_XSSSSM: case K_XLARFB: case K_XSSRFB:
      return ssrfb_reg_ok(b, ib) ? b / NSR : ceil_div(b, NS);  // slabs
    case K_XTRSMU: case K_XUNSSSSM: case K_XUNGESSM: return ceil_div(b, 32);
    case K_XGEMM: return ceil_div(b, 64);
    default: return 1;                 // panels, RECV
  }
}

// SEND: j = offset into Dist::sends, pad = producer kind, nitems = npeers * SEND_CHUNKS.
struct TaskD {
  int kind, k, i, j;
  int nitems, item0, level, pad;
};

struct Prob {
  double* A;
  double* aux;   // T strips (QR) / L strips (LU)
  int* ipiv;
  double* vx;    // explicit unit-lower V_kk / L_kk copies, p tiles of b*b
  double* scratch;
  size_t scr_stride;
  int n, b, ib, p;
  int* info;     // INT_MAX = no failure (rank-local accumulator in multi-GPU mode)
  double* X;     // solve / apply DAGs: right-hand sides in BDL, p x q tiles (tile (i,c) at (i + c*p)*b*b)
  int q;
  int nopiv;     // LU without pivoting (GENP)
};

struct Sched {
  const TaskD* tasks;
  const int* succ_off;
  const int* succ;
  const int* item_task;
  int ntasks, nitems;
  int qbase[NLEV + 1];
  int* indeg;
  int* items_done;
  int* q;
  int* head;   // [NLEV]
  int* tail;   // [NLEV]
  int* ndone;
  int* abort_flag;
  int* exit_count;
  long long* trace;  // 5 per item or null
  int trace_cap;
  // copy overlap (0 / null unless the DAG has ARRIVE / DONE tasks)
  const int* arrive_flags;  // [narrive], set to 1 by the H2D copy stream after tile column j
  int* arrive_next;         // next column whose ARRIVE task is still pending
  int arrive_task0, narrive;
  int* done_flags;          // [narrive], set to 1 by DONE(j)
};

// One remote push: when a SEND task completes, item `item` (the consumer's RECV task)
// is appended to level `level` of rank `peer`'s queue (queue region starts at qbase).
struct SendEnt {
  int peer, item, level, qbase, qcap;  // qcap: end of that level's queue region (checks)
};

// Symmetric per-rank block ("sym"), identical offsets on every rank:
//   [sync ints][sched state ints][queue ints][cache tiles][cache strips][cache ipiv]
// SY_PROBE[r] / SY_PROBE_CNT: written by peers' tile_dist_probe (IPC path check, no waiting)
enum SyncSlot { SY_ARRIVE = 0, SY_DEPART = 8, SY_INFO = 16, SY_GO = 24, SY_ABORT = 25, SY_LINFO = 26,
                SY_PROBE = 32, SY_PROBE_CNT = 40, SY_INTS = 48 };

struct Dist {
  int nranks;        // 0 = single-GPU mode (direct BDL addressing, no barriers)
  int rank;
  int epoch;         // call counter, identical on every rank (barrier tag)
  int cta0, nctas;   // this rank's CTA range in the grid
  double* const* tptr;  // [p*p] tile (i,j) -> local storage or receive-cache slot (or null)
  double* const* sptr;  // [p*p] T / L strip (i,k)
  int* const* pptr;     // [p*p] ipiv vector (i,k)
  double* const* vptr;  // [p]   explicit V_kk / L_kk copy
  const SendEnt* sends;
  char* peer_sym[TF_MAX_RANKS];  // every rank's sym block (peer-mapped; own included)
  size_t off_tail, off_q, off_ctile, off_cstrip, off_cpiv;  // byte offsets inside sym
  size_t sym_bytes;
  int* user_info;    // caller's d_info (written once at the end)
  long long timeout_ns;
};

struct RankRun {
  Prob P;
  Sched S;
  Dist D;
};

struct Runs {
  int nruns;
  RankRun r[TF_MAX_RANKS];
};

// receive-cache slot of panel tile (i,k), i >= k (packed lower triangle, column k major)
TF_HD inline long long cache_slot(int i, int k, int p) {
  return (long long)k * p - (long long)k * (k - 1) / 2 + (i - k);
}

// launch wrappers (tf_device.cu)
int launch_sched_reset(const Sched& S, const int* indeg0, int qtotal, int* info, void* stream);
int launch_sched_seed(const Sched& S, const int* roots, int nroots, void* stream);
int launch_persistent(const Runs& R, int ctas, size_t smem, void* stream, bool coop);
int launch_tk(int kind, int b, int ib, double* t0, double* t1, double* t2, double* aux, int* ipiv, double* vx,
              double* scratch, size_t scr_stride, int* info, int items, size_t smem, void* stream);
int launch_unit_lower(const double* A, double* X, int b, void* stream);
int launch_pack(int64_t m, int64_t n, int64_t b, double* D, double* T, int dir, void* stream);
int launch_probe(char* peer_sym, int rank, int value, void* stream);
int launch_xpack(int64_t n, int64_t nrhs, int64_t ldx, int64_t b, int64_t q, double* X, double* T, int dir,
                 void* stream);
int device_kernel_setup(size_t smem);
int tk_kernel_setup(size_t smem);
size_t smem_bytes();

}  // namespace tf
