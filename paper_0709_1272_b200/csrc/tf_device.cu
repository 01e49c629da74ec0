// tf_device.cu — device side of libtilefact.so: the persistent DAG scheduler kernel, the
// multi-GPU SEND/RECV work items and barriers, the per-kernel test launcher, layout
// kernels, and the launch wrappers declared in tf_sched.h.
//
// Execution model ("Graph driven asynchronous execution"): the
// implicit DAG of Algorithms 1-3 (built on the host, tf_host.cpp) is executed by ONE
// persistent kernel per factorization: every CTA (one per SM) repeatedly pops the
// highest-priority ready work item from global-memory queues, runs the tile kernel, and
// on the last item of a task decrements its successors' dependency counters, pushing
// those that become ready.  This is the paper's self-scheduled progress-table runtime
// moved onto the GPU: no host round trip, no kernel launch per task.
//
// Multi-GPU: the same kernel runs one rank's local DAG.  A SEND task's
// items store the producer's panel tile (and T strip / pivots) straight into each
// consumer rank's receive cache over NVLink; its last item then pushes the consumer's
// RECV task into that rank's ready queue with remote atomics (device-initiated, no host
// proxy).  Several ranks can share one launch (CTA groups) — that is how the multi-rank
// path runs on a single GPU; with one rank per GPU the peers are IPC-mapped.
#include <cuda_runtime.h>

#include <climits>

// Every tile-kernel variant is its own (noinline) function with its own register
// allocation; the persistent kernel's scheduler loop calls them (tf_kernels.cuh).
#define TF_SPLIT_ITEMS
#include "tf_kernels.cuh"
#include "tf_sched.h"

namespace tf {

// TF_CHECK builds (tools/, debugging only): bounds / null checks that trap with a message.
#ifdef TF_CHECK
#define TF_ASSERT(cond, ...)                                      \
  do {                                                            \
    if (!(cond)) {                                                \
      printf("TF_ASSERT %s:%d: ", __FILE__, __LINE__);            \
      printf(__VA_ARGS__);                                        \
      printf("\n");                                               \
      __trap();                                                   \
    }                                                             \
  } while (0)
#else
#define TF_ASSERT(cond, ...) \
  do {                       \
  } while (0)
#endif

__device__ __forceinline__ int ld_volatile(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(int* p, int v) {
  asm volatile("st.relaxed.sys.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

// acquire-release fences (lighter than the sequentially consistent __threadfence*(); a
// gpu-scope fence still invalidates L1, B300_MICROARCH: CCTL.IVALL for scope >= cluster)
__device__ __forceinline__ void fence_ar_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ void fence_ar_sys() { asm volatile("fence.acq_rel.sys;\n" ::: "memory"); }

__device__ __forceinline__ int* sym_sync(const Dist& D, int r) { return reinterpret_cast<int*>(D.peer_sym[r]); }

// Set the abort flag of every rank (Cholesky failure, or a multi-GPU timeout).
__device__ inline void abort_all(const Sched& S, const Dist& D) {
  atomicExch(S.abort_flag, 1);
  for (int r = 0; r < D.nranks; ++r) st_release_sys(sym_sync(D, r) + SY_ABORT, 1);
}

__device__ inline void sched_push(const Sched& S, int s) {
  const TaskD d = S.tasks[s];
  const int slot = atomicAdd(&S.tail[d.level], d.nitems);
  volatile int* q = S.q + S.qbase[d.level] + slot;
  for (int x = 0; x < d.nitems; ++x) q[x] = d.item0 + x;
}

// Completion of task t by a single thread (the scheduler's ARRIVE tasks): successors'
// counters decremented, ready ones pushed, the task counted.
__device__ inline void complete_task_single(const Sched& S, int t) {
  fence_ar_gpu();
  for (int e = S.succ_off[t]; e < S.succ_off[t + 1]; ++e) {
    const int s = S.succ[e];
    if (atomicSub(&S.indeg[s], 1) == 1) {
      fence_ar_gpu();
      sched_push(S, s);
    }
  }
  fence_ar_gpu();
  atomicAdd(S.ndone, 1);
}

// Copy overlap: if the next pending tile column has arrived (its flag was written by the
// H2D copy stream after the column's data), complete its ARRIVE task.  One poller wins the
// column by CAS.  Returns true if a column was released.
__device__ inline bool poll_arrivals(const Sched& S) {
  if (S.narrive == 0) return false;
  const int j = ld_volatile(S.arrive_next);
  if (j >= S.narrive || ld_acquire_sys(S.arrive_flags + j) == 0) return false;
  if (atomicCAS(S.arrive_next, j, j + 1) != j) return false;
  fence_ar_sys();  // the column's bytes (copy engine) before the tasks that read them
  complete_task_single(S, S.arrive_task0 + j);
  return true;
}

// Pop the next item: highest non-empty level first, FIFO inside a level.
// Returns item id, -1 when every task has completed, -2 on abort.
__device__ inline int sched_pop(const Sched& S, const Dist& D, int* info) {
  long long idle0 = 0;
  for (;;) {
    if (ld_volatile(S.abort_flag)) return -2;
    bool retry = false;
    // all heads and tails in two vector loads (one L2 round trip instead of 2*NLEV)
    int hv[NLEV], tv[NLEV];
    asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(hv[0]), "=r"(hv[1]), "=r"(hv[2]), "=r"(hv[3]) : "l"(S.head) : "memory");
    asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(tv[0]), "=r"(tv[1]), "=r"(tv[2]), "=r"(tv[3]) : "l"(S.tail) : "memory");
    for (int lev = 0; lev < NLEV; ++lev) {
      const int h = hv[lev];
      const int t = tv[lev];
      if (h < t) {
        // With a backlog of at least two items per CTA nobody can over-claim, so the head is
        // taken by an unconditional fetch-add: no CAS retry round trips when many CTAs finish
        // equal items at the same moment (every CTA holds at most one claim at a time).
        int hh = h;
        bool got;
        if (t - h >= 2 * (int)gridDim.x) {
          hh = atomicAdd(&S.head[lev], 1);
          got = true;
        } else {
          got = atomicCAS(&S.head[lev], h, h + 1) == h;
        }
        if (got) {
          const volatile int* slot = S.q + S.qbase[lev] + hh;
          int v;
          while ((v = *slot) < 0) {
          }
          TF_ASSERT(v < S.nitems, "popped item %d >= nitems %d (level %d slot %d)", v, S.nitems, lev, hh);
          // acquire: the producers' tile writes are visible (and L1 is invalidated); peer
          // GPUs' stores into the receive cache need the system-scope fence
          if (D.nranks > 1) fence_ar_sys();
          else fence_ar_gpu();
          fence_proxy_async_all();  // ... also to this thread's bulk (async-proxy) copies
          return v;
        }
        retry = true;
        break;
      }
    }
    if (!retry) {
      if (ld_volatile(S.ndone) >= S.ntasks) return -1;
      if (poll_arrivals(S)) { idle0 = 0; continue; }
      if (D.timeout_ns > 0) {
        const long long now = globaltimer();
        if (idle0 == 0) idle0 = now;
        else if (now - idle0 > D.timeout_ns) {
          atomicExch(info, -1);
          abort_all(S, D);
          return -2;
        }
      }
      __nanosleep(32);
    }
  }
}

// Remote push of a consumer rank's RECV item (one SendEnt).
__device__ inline void remote_push(const Dist& D, const SendEnt& e) {
  char* sym = D.peer_sym[e.peer];
  int* tail = reinterpret_cast<int*>(sym + D.off_tail);
  int* q = reinterpret_cast<int*>(sym + D.off_q);
  const int slot = atomicAdd_system(&tail[e.level], 1);
  TF_ASSERT(e.qbase + slot < e.qcap, "remote queue overflow peer %d level %d slot %d", e.peer, e.level, slot);
  st_release_sys(q + e.qbase + slot, e.item);
}

// Completion of item `it` by one whole warp (overlapping the next pop by thread 0): lane 0
// releases the CTA's writes (the preceding __syncthreads makes them cumulative) and counts
// the item; if it was the task's last item, the lanes decrement the successors' counters in
// parallel and push the ready ones, and lane 0 counts the task.
__device__ inline void sched_complete_warp(const Sched& S, const Dist& D, int it) {
  const int lane = threadIdx.x & 31;
  const int t = S.item_task[it];
  int last = 0;
  if (lane == 0) {
    if (D.nranks > 1) fence_ar_sys();  // release this item's (peer) writes
    else fence_ar_gpu();
    last = atomicAdd(&S.items_done[t], 1) == S.tasks[t].nitems - 1;
    if (last) fence_ar_gpu();  // acquire the other items' writes
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  __syncwarp();
  if (!last) return;
  const TaskD d = S.tasks[t];
  if (d.kind == K_SEND) {
    fence_ar_sys();  // the other items' peer stores, released to the peers
    const int npeers = d.nitems / SEND_CHUNKS;
    for (int x = lane; x < npeers; x += 32) remote_push(D, D.sends[d.j + x]);
  }
  fence_ar_gpu();
  for (int e = S.succ_off[t] + lane; e < S.succ_off[t + 1]; e += 32) {
    const int s = S.succ[e];
    if (atomicSub(&S.indeg[s], 1) == 1) {
      fence_ar_gpu();
      sched_push(S, s);
    }
  }
  __syncwarp();
  if (lane == 0) {
    fence_ar_gpu();
    atomicAdd(S.ndone, 1);
  }
}

// ------------------------------------------------------------------ tile addressing
struct Addr {
  const Prob& P;
  const Dist& D;
  __device__ Addr(const Prob& p, const Dist& d) : P(p), D(d) {}
  __device__ double* T(int i, int j) const {
    TF_ASSERT(i >= 0 && j >= 0 && i < P.p && j < P.p, "T(%d,%d) p=%d", i, j, P.p);
    TF_ASSERT(!D.tptr || D.tptr[i + (size_t)j * P.p], "rank %d: null tile (%d,%d)", D.rank, i, j);
    if (D.tptr) return D.tptr[i + (size_t)j * P.p];
    return P.A + ((size_t)i + (size_t)j * P.p) * (size_t)P.b * P.b;
  }
  __device__ double* STRIP(int i, int k) const {
    TF_ASSERT(!D.sptr || D.sptr[i + (size_t)k * P.p], "rank %d: null strip (%d,%d)", D.rank, i, k);
    if (D.sptr) return D.sptr[i + (size_t)k * P.p];
    return P.aux + ((size_t)i + (size_t)k * P.p) * (size_t)P.ib * P.b;
  }
  __device__ int* PIV(int i, int k) const {
    TF_ASSERT(!D.pptr || D.pptr[i + (size_t)k * P.p], "rank %d: null ipiv (%d,%d)", D.rank, i, k);
    if (D.pptr) return D.pptr[i + (size_t)k * P.p];
    return P.ipiv + ((size_t)i + (size_t)k * P.p) * P.b;
  }
  __device__ double* X(int i, int c) const { return P.X + ((size_t)i + (size_t)c * P.p) * (size_t)P.b * P.b; }
  __device__ double* VX(int k) const {
    TF_ASSERT(!D.vptr || D.vptr[k], "rank %d: null VX(%d)", D.rank, k);
    if (D.vptr) return D.vptr[k];
    return P.vx + (size_t)k * P.b * P.b;
  }
};

// SEND item: chunk c of the payload produced by task (pad, k, i) to peer #pe of the list.
// Payload (what the consumers read):
//   POTRF(k): L_kk        TRSM(i,k): L_ik
//   GEQRT(k): V_kk copy + T strip (k,k)      TSQRT(i,k): V_ik + T strip (i,k)
//   GETRF(k): L_kk copy + ipiv (k,k)         TSTRF(i,k): L_ik + L strip (i,k) + ipiv (i,k)
// Destination: the same slots of the peer's receive cache (cache_slot(i,k)).
__device__ inline void send_item(const Addr& a, const TaskD& d, int sub) {
  const Prob& P = a.P;
  const Dist& D = a.D;
  const int pe = sub / SEND_CHUNKS, c = sub % SEND_CHUNKS;
  const SendEnt e = D.sends[d.j + pe];
  TF_ASSERT(e.peer >= 0 && e.peer < D.nranks && e.peer != D.rank, "bad peer %d", e.peer);
  char* sym = D.peer_sym[e.peer];
  const size_t bb8 = (size_t)P.b * P.b * 8, sb8 = (size_t)P.ib * P.b * 8, pb4 = (size_t)P.b * 4;
  const int pk = d.pad, k = d.k, i = d.i;
  const long long slot = cache_slot(i, k, P.p);
  const char* src[3];
  char* dst[3];
  size_t len[3];
  int ns = 0;
  auto add = [&](const void* s, size_t off, size_t bytes) {
    src[ns] = reinterpret_cast<const char*>(s);
    dst[ns] = sym + off;
    len[ns] = bytes;
    ++ns;
  };
  switch (pk) {
    case 0: add(a.T(k, k), D.off_ctile + slot * bb8, bb8); break;
    case 1: add(a.T(i, k), D.off_ctile + slot * bb8, bb8); break;
    case 4: add(a.VX(k), D.off_ctile + slot * bb8, bb8); add(a.STRIP(k, k), D.off_cstrip + slot * sb8, sb8); break;
    case 6: add(a.T(i, k), D.off_ctile + slot * bb8, bb8); add(a.STRIP(i, k), D.off_cstrip + slot * sb8, sb8); break;
    case 8: add(a.VX(k), D.off_ctile + slot * bb8, bb8); add(a.PIV(k, k), D.off_cpiv + slot * pb4, pb4); break;
    case 10:
      add(a.T(i, k), D.off_ctile + slot * bb8, bb8);
      add(a.STRIP(i, k), D.off_cstrip + slot * sb8, sb8);
      add(a.PIV(i, k), D.off_cpiv + slot * pb4, pb4);
      break;
    default: return;
  }
  size_t total = 0;
  for (int s = 0; s < ns; ++s) {
    total += len[s];
    TF_ASSERT((size_t)(dst[s] - sym) + len[s] <= D.sym_bytes, "send dst overflow seg %d slot %lld", s, slot);
  }
  const size_t nvec = total / 16;  // every segment is a multiple of 16 bytes (b % 4 == 0)
  const size_t lo = nvec * c / SEND_CHUNKS * 16, hi = nvec * (c + 1) / SEND_CHUNKS * 16;
  size_t base = 0;
  for (int s = 0; s < ns; ++s) {
    // this chunk's byte range [lo, hi) intersected with segment s = [base, base + len)
    const size_t g0 = lo > base ? lo : base, g1 = hi < base + len[s] ? hi : base + len[s];
    if (g0 < g1) {
      const size_t a0 = g0 - base, a1 = g1 - base;
      const int4* sp = reinterpret_cast<const int4*>(src[s] + a0);
      int4* dp = reinterpret_cast<int4*>(dst[s] + a0);
      const size_t nv = (a1 - a0) / 16;
      size_t x = threadIdx.x;
      for (; x + 3 * TF_THREADS < nv; x += 4 * TF_THREADS) {
        const int4 v0 = __ldcg(sp + x), v1 = __ldcg(sp + x + TF_THREADS), v2 = __ldcg(sp + x + 2 * TF_THREADS),
                   v3 = __ldcg(sp + x + 3 * TF_THREADS);
        dp[x] = v0;
        dp[x + TF_THREADS] = v1;
        dp[x + 2 * TF_THREADS] = v2;
        dp[x + 3 * TF_THREADS] = v3;
      }
      for (; x < nv; x += TF_THREADS) dp[x] = __ldcg(sp + x);
    }
    base += len[s];
  }
}

// Dispatch one work item to its tile kernel.
__device__ inline void run_item(const Prob& P, const Sched& S, const Dist& D, const TaskD& d, int sub, Ctx& cx,
                                double* sm) {
  const Addr a(P, D);
  const int k = d.k, i = d.i, j = d.j;
  switch (d.kind) {
    case 0: {
      const int f = potrf_item(cx, a.T(k, k), sm);
      if (f >= 0 && threadIdx.x == 0) {
        atomicMin(cx.info, k * P.b + f + 1);
        if (D.nranks > 1) abort_all(S, D);
        else atomicExch(cx.abort_flag, 1);
      }
    } break;
    case 1: trsm_item(cx, a.T(k, k), a.T(i, k), sub, sm); break;
    case 2: syrk_item(cx, a.T(i, k), a.T(i, i), sub, sm); break;
    case 3:
      if (d.pad) v_gemm_tile(cx, a.T(i, k), a.T(j, k), a.T(i, j));  // whole tile as one item (panel-level graph)
      else gemm_item(cx, a.T(i, k), a.T(j, k), a.T(i, j), sub, sm);
      break;
    case 4: geqrt_item(cx, a.T(k, k), a.STRIP(k, k), a.VX(k), sm); break;
    case 5: larfb_item(cx, a.VX(k), a.STRIP(k, k), a.T(k, j), sub + d.pad, sm); break;
    case 6: tsqrt_item(cx, a.T(k, k), a.T(i, k), a.STRIP(i, k), sm); break;
    case 7: ssrfb_item(cx, a.T(i, k), a.STRIP(i, k), a.T(k, j), a.T(i, j), sub + d.pad, sm); break;
    case 8: {
      const int f = getrf_item(cx, a.T(k, k), a.PIV(k, k), a.VX(k), sm);
      if (f >= 0 && threadIdx.x == 0) atomicMin(cx.info, k * P.b + f + 1);
    } break;
    case 9: gessm_item(cx, a.VX(k), a.PIV(k, k), a.T(k, j), sub + d.pad, sm); break;
    case 10: {
      const int f = tstrf_item(cx, a.T(k, k), a.T(i, k), a.STRIP(i, k), a.PIV(i, k), sm);
      if (f >= 0 && threadIdx.x == 0) atomicMin(cx.info, k * P.b + f + 1);
    } break;
    case 11: ssssm_item(cx, a.T(i, k), a.STRIP(i, k), a.PIV(i, k), a.T(k, j), a.T(i, j), sub + d.pad, sm); break;
    // panel-level Cholesky DAG (d.pad = 128-column panel)
    case K_POTRF_D: {
      const int f = v_potrf_pd(cx, a.T(k, k), d.pad);
      if (f >= 0 && threadIdx.x == 0) {
        atomicMin(cx.info, k * P.b + f + 1);
        atomicExch(cx.abort_flag, 1);
      }
    } break;
    case K_POTRF_B: v_potrf_pb(cx, a.T(k, k), d.pad, sub); break;
    case K_TRSM_P: v_trsm_p(cx, a.T(k, k), a.T(i, k), d.pad, sub); break;
    // slab-level DAG panel tasks (d.pad = slab)
    case K_GEQRT_S: geqrt_slab_item(cx, a.T(k, k), a.STRIP(k, k), a.VX(k), d.pad, sm); break;
    case K_TSQRT_S: tsqrt_slab_item(cx, a.T(k, k), a.T(i, k), a.STRIP(i, k), d.pad, sm); break;
    case K_TSTRF_A: tstrf_apply_item(cx, a.T(k, k), a.T(i, k), a.STRIP(i, k), a.PIV(i, k), d.pad, sm); break;
    case K_GETRF_S: {
      const int f = getrf_slab_item(cx, a.T(k, k), a.PIV(k, k), a.VX(k), d.pad, sm);
      if (f >= 0 && threadIdx.x == 0) atomicMin(cx.info, k * P.b + f + 1);
    } break;
    case K_TSTRF_S: {
      const int f = tstrf_slab_item(cx, a.T(k, k), a.T(i, k), a.STRIP(i, k), a.PIV(i, k), d.pad, sm);
      if (f >= 0 && threadIdx.x == 0) atomicMin(cx.info, k * P.b + f + 1);
    } break;
    // solve / apply tasks (tf_solve.cuh); d.j = the right-hand-side tile column c
    case K_UNITL: unitl_item(cx, a.T(k, k), a.VX(k)); break;
    case K_XGESSM: gessm_item(cx, a.VX(k), a.PIV(k, k), a.X(k, j), sub, sm); break;
    case K_XSSSSM: ssssm_item(cx, a.T(i, k), a.STRIP(i, k), a.PIV(i, k), a.X(k, j), a.X(i, j), sub, sm); break;
    case K_XLARFB: larfb_item(cx, a.VX(k), a.STRIP(k, k), a.X(k, j), sub, sm); break;
    case K_XSSRFB: ssrfb_item(cx, a.T(i, k), a.STRIP(i, k), a.X(k, j), a.X(i, j), sub, sm); break;
    case K_XTRSMU: v_trsmu(cx, a.T(k, k), a.X(k, j), sub); break;
    case K_XGEMM: v_xgemm(cx, a.T(i, k), a.X(k, j), a.X(i, j), sub); break;
    case K_XUNSSSSM: v_unssssm(cx, a.T(i, k), a.STRIP(i, k), a.PIV(i, k), a.X(k, j), a.X(i, j), sub); break;
    case K_XUNGESSM: v_ungessm(cx, a.T(k, k), a.PIV(k, k), a.X(k, j), sub); break;
    case K_DONE:  // every tile of column d.j is final: release the D2H copy of that column
      if (threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys(S.done_flags + d.j, 1);
      }
      break;
    case K_SEND: send_item(a, d, sub); break;
    case K_RECV: break;  // the data is already in the cache; completing releases the consumers
    default: break;
  }
}

// Wait until slot[r] of this rank's sync block reaches `epoch` for every rank r.
// Returns false on timeout.
__device__ inline bool wait_all(const Dist& D, int slot0) {
  const int* me = sym_sync(D, D.rank);
  const long long t0 = globaltimer();
  for (int r = 0; r < D.nranks; ++r) {
    while (ld_acquire_sys(me + slot0 + r) - D.epoch < 0) {
      if (D.timeout_ns > 0 && globaltimer() - t0 > D.timeout_ns) return false;
      __nanosleep(64);
    }
  }
  return true;
}

__global__ void __launch_bounds__(TF_THREADS, 1) tf_persistent(const __grid_constant__ Runs R) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_it;
  int rk = 0;
  for (int r = 1; r < R.nruns; ++r)
    if ((int)blockIdx.x >= R.r[r].D.cta0) rk = r;
  const Prob& P = R.r[rk].P;
  const Sched& S = R.r[rk].S;
  const Dist& D = R.r[rk].D;
  Ctx cx;
  cx.b = P.b;
  cx.ib = P.ib;
  cx.scratch = P.scratch + (size_t)(blockIdx.x - D.cta0) * P.scr_stride;
  cx.info = P.info;
  cx.abort_flag = S.abort_flag;
  cx.nopiv = P.nopiv;
  pipe_init(sm);
  if (D.nranks > 0) {
    // start barrier: no peer may push into this rank's queues before it has been reset
    int* me = sym_sync(D, D.rank);
    if (threadIdx.x == 0) {
      if ((int)blockIdx.x == D.cta0) {
        for (int r = 0; r < D.nranks; ++r) st_release_sys(sym_sync(D, r) + SY_ARRIVE + D.rank, D.epoch);
        if (!wait_all(D, SY_ARRIVE)) {
          atomicExch(P.info, -1);
          abort_all(S, D);
        }
        st_release_sys(me + SY_GO, D.epoch);
      } else {
        // the same protocol timeout as wait_all: a leader that never arrives becomes
        // info = -1 and an abort, not a hung GPU
        const long long t0 = globaltimer();
        while (ld_acquire_sys(me + SY_GO) - D.epoch < 0) {
          if (D.timeout_ns > 0 && globaltimer() - t0 > D.timeout_ns) {
            atomicExch(P.info, -1);
            atomicExch(S.abort_flag, 1);
            break;
          }
          __nanosleep(64);
        }
      }
    }
    __syncthreads();
  }
  // Thread 0 pops the next item while warp 1 completes the previous one: the scheduler
  // round trips of the two overlap instead of adding up between items.
  int prev = -1;
  for (;;) {
    if (threadIdx.x == 0) s_it = sched_pop(S, D, P.info);
    else if ((threadIdx.x >> 5) == 1 && prev >= 0) sched_complete_warp(S, D, prev);
    __syncthreads();
    const int it = s_it;
    if (it < 0) break;
    const int t = S.item_task[it];
    const TaskD d = S.tasks[t];
    TF_ASSERT(it - d.item0 >= 0 && it - d.item0 < d.nitems, "item %d outside task %d", it, t);
    const long long t0 = S.trace ? globaltimer() : 0;
    run_item(P, S, D, d, it - d.item0, cx, sm);
    __syncthreads();
    if (threadIdx.x == 0 && S.trace && it < S.trace_cap) {
      long long* r = S.trace + (size_t)it * 5;
      r[0] = t;
      r[1] = it - d.item0;
      r[2] = smid();
      r[3] = t0;
      r[4] = globaltimer();
    }
    prev = it;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const int nct = D.nranks > 0 ? D.nctas : (int)gridDim.x;
    if (atomicAdd(S.exit_count, 1) == nct - 1) {
      if (D.nranks == 0) {
        if (ld_volatile(P.info) == INT_MAX) *P.info = 0;
      } else {
        // end barrier: every peer has finished (so no more stores or pushes target this
        // rank), and the info values of all ranks are combined (-1 = timeout, else min)
        const int li = ld_volatile(P.info);
        for (int r = 0; r < D.nranks; ++r) st_relaxed_sys(sym_sync(D, r) + SY_INFO + D.rank, li);
        __threadfence_system();
        for (int r = 0; r < D.nranks; ++r) st_release_sys(sym_sync(D, r) + SY_DEPART + D.rank, D.epoch);
        int res = INT_MAX;
        if (!wait_all(D, SY_DEPART)) {
          res = -1;
        } else {
          const int* me = sym_sync(D, D.rank);
          for (int r = 0; r < D.nranks; ++r) {
            const int v = ld_volatile(me + SY_INFO + r);
            if (v == -1 || res == -1) res = -1;
            else if (v < res) res = v;
          }
        }
        if (D.user_info) *D.user_info = (res == INT_MAX) ? 0 : res;
      }
    }
  }
}

__global__ void tf_sched_reset(Sched S, const int* indeg0, int qtotal, int* info) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int t = tid; t < S.ntasks; t += nth) {
    S.indeg[t] = indeg0[t];
    S.items_done[t] = 0;
  }
  for (int x = tid; x < qtotal; x += nth) S.q[x] = -1;
  if (tid < NLEV) { S.head[tid] = 0; S.tail[tid] = 0; }
  if (tid == 0) {
    *S.ndone = 0;
    *S.abort_flag = 0;
    *S.exit_count = 0;
    *info = INT_MAX;
  }
}

__global__ void tf_sched_seed(Sched S, const int* roots, int nroots) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int r = 0; r < nroots; ++r) sched_push(S, roots[r]);
}

__global__ void pack_kernel(int64_t m, int64_t n, int64_t b, double* D, double* T, int dir) {
  const int64_t p = m / b;
  const int64_t tot = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    // e indexes the tile storage: tile t = e / b^2, within-tile offset w
    const int64_t bb = b * b;
    const int64_t t = e / bb, w = e % bb;
    const int64_t ti = t % p, tj = t / p;
    const int64_t r = ti * b + w % b, c = tj * b + w / b;
    if (dir == 0) T[e] = D[r + c * m];
    else D[r + c * m] = T[e];
  }
}

// Right-hand sides: dense column-major X (n x nrhs, ld ldx) <-> BDL tiles of an n x q*b
// matrix (tile (i,c) at (i + c*p)*b*b), padding columns >= nrhs with zeros.
__global__ void xpack_kernel(int64_t n, int64_t nrhs, int64_t ldx, int64_t b, int64_t q, double* X, double* T,
                             int dir) {
  const int64_t p = n / b, bb = b * b, tot = n * q * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / bb, w = e % bb;
    const int64_t r = (t % p) * b + w % b, c = (t / p) * b + w / b;
    if (dir == 0) T[e] = c < nrhs ? X[r + c * ldx] : 0.0;
    else if (c < nrhs) X[r + c * ldx] = T[e];
  }
}

// IPC path check (tile_dist_probe): one system-scope release store of `value` into the
// peer's probe slot for this rank and one system-scope atomic on its probe counter.
__global__ void probe_kernel(int* peer_sync, int rank, int value) {
  if (threadIdx.x == 0) {
    st_release_sys(peer_sync + SY_PROBE + rank, value);
    atomicAdd_system(peer_sync + SY_PROBE_CNT, 1);
  }
}

// ------------------------------------------------------------------ launch wrappers
size_t smem_bytes() { return (size_t)SMEM_DOUBLES * sizeof(double); }

static int ok_or(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

int device_kernel_setup(size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(tf_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  return tk_kernel_setup(smem);
}

int launch_sched_reset(const Sched& S, const int* indeg0, int qtotal, int* info, void* stream) {
  tf_sched_reset<<<64, 256, 0, (cudaStream_t)stream>>>(S, indeg0, qtotal, info);
  return ok_or(cudaGetLastError());
}
int launch_sched_seed(const Sched& S, const int* roots, int nroots, void* stream) {
  tf_sched_seed<<<1, 32, 0, (cudaStream_t)stream>>>(S, roots, nroots);
  return ok_or(cudaGetLastError());
}
// coop: cooperative launch (all CTAs guaranteed co-resident or the launch fails), used
// whenever CTAs wait on one another (multi-rank barriers, emulated ranks).
int launch_persistent(const Runs& R, int ctas, size_t smem, void* stream, bool coop) {
  if (!coop) {
    tf_persistent<<<ctas, TF_THREADS, smem, (cudaStream_t)stream>>>(R);
    return ok_or(cudaGetLastError());
  }
  void* args[] = {const_cast<Runs*>(&R)};
  return ok_or(cudaLaunchCooperativeKernel((const void*)tf_persistent, dim3(ctas), dim3(TF_THREADS), args, smem,
                                           (cudaStream_t)stream));
}
int launch_probe(char* peer_sym, int rank, int value, void* stream) {
  probe_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<int*>(peer_sym), rank, value);
  return ok_or(cudaGetLastError());
}
int launch_xpack(int64_t n, int64_t nrhs, int64_t ldx, int64_t b, int64_t q, double* X, double* T, int dir,
                 void* stream) {
  xpack_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(n, nrhs, ldx, b, q, X, T, dir);
  return ok_or(cudaGetLastError());
}
int launch_pack(int64_t m, int64_t n, int64_t b, double* D, double* T, int dir, void* stream) {
  pack_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(m, n, b, D, T, dir);
  return ok_or(cudaGetLastError());
}

}  // namespace tf
