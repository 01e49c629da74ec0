// tf_lib.cu — libtilefact.so: the persistent device-side DAG scheduler, the host task-graph
// builder, workspace caches and the C-ABI declared in include/tilefact.h.
//
// Execution model ("Graph driven asynchronous execution"): the
// implicit DAG of Algorithms 1-3 is built once on the host per (algorithm, p, b, policy)
// with the dependency rules of SURVEY.md §8(a) a13 (diagonal tiles tracked as two
// regions, V/L vs R/U), uploaded, and executed by ONE persistent kernel per
// factorization: every CTA (one per SM) repeatedly pops the highest-priority ready work
// item from global-memory queues, runs the tile kernel, and on the last item of a task
// decrements its successors' dependency counters, pushing those that become ready.
// This is the paper's self-scheduled progress-table runtime moved
// onto the GPU: no host round trip, no kernel launch per task.
#include <cuda_runtime.h>

#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/tilefact.h"
#include "tf_kernels.cuh"

namespace tf {

constexpr int NLEV = 4;

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
  int* info;
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
};

__device__ __forceinline__ int ld_volatile(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

__device__ inline void sched_push(const Sched& S, int s) {
  const TaskD d = S.tasks[s];
  const int slot = atomicAdd(&S.tail[d.level], d.nitems);
  volatile int* q = S.q + S.qbase[d.level] + slot;
  for (int x = 0; x < d.nitems; ++x) q[x] = d.item0 + x;
}

// Pop the next item: highest non-empty level first, FIFO inside a level.
// Returns item id, -1 when every task has completed, -2 on abort.
__device__ inline int sched_pop(const Sched& S) {
  for (;;) {
    if (ld_volatile(S.abort_flag)) return -2;
    bool retry = false;
    for (int lev = 0; lev < NLEV; ++lev) {
      const int h = ld_volatile(&S.head[lev]);
      const int t = ld_volatile(&S.tail[lev]);
      if (h < t) {
        if (atomicCAS(&S.head[lev], h, h + 1) == h) {
          const volatile int* slot = S.q + S.qbase[lev] + h;
          int v;
          while ((v = *slot) < 0) {
          }
          __threadfence();         // acquire: the producers' tile writes are visible (and L1 is invalidated)
          fence_proxy_async_all();  // ... also to this thread's bulk (async-proxy) copies
          return v;
        }
        retry = true;
        break;
      }
    }
    if (!retry) {
      if (ld_volatile(S.ndone) >= S.ntasks) return -1;
      __nanosleep(32);
    }
  }
}

__device__ inline void sched_complete(const Sched& S, int it) {
  const int t = S.item_task[it];
  __threadfence();  // release this item's writes
  if (atomicAdd(&S.items_done[t], 1) == S.tasks[t].nitems - 1) {
    __threadfence();  // acquire the other items' writes before releasing successors
    for (int e = S.succ_off[t]; e < S.succ_off[t + 1]; ++e) {
      const int s = S.succ[e];
      if (atomicSub(&S.indeg[s], 1) == 1) {
        __threadfence();
        sched_push(S, s);
      }
    }
    __threadfence();
    atomicAdd(S.ndone, 1);
  }
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

// Dispatch one work item to its tile kernel.
__device__ inline void run_item(const Prob& P, const TaskD& d, int sub, Ctx& cx, double* sm) {
  const size_t bb = (size_t)P.b * P.b;
  auto T = [&](int i, int j) { return P.A + ((size_t)i + (size_t)j * P.p) * bb; };
  auto STRIP = [&](int i, int k) { return P.aux + ((size_t)i + (size_t)k * P.p) * (size_t)P.ib * P.b; };
  auto PIV = [&](int i, int k) { return P.ipiv + ((size_t)i + (size_t)k * P.p) * P.b; };
  auto VX = [&](int k) { return P.vx + (size_t)k * bb; };
  const int k = d.k, i = d.i, j = d.j;
  switch (d.kind) {
    case 0: {
      const int f = potrf_item(cx, T(k, k), sm);
      if (f >= 0 && threadIdx.x == 0) {
        atomicMin(cx.info, k * P.b + f + 1);
        atomicExch(cx.abort_flag, 1);
      }
    } break;
    case 1: trsm_item(cx, T(k, k), T(i, k), sub, sm); break;
    case 2: syrk_item(cx, T(i, k), T(i, i), sub, sm); break;
    case 3: gemm_item(cx, T(i, k), T(j, k), T(i, j), sub, sm); break;
    case 4: geqrt_item(cx, T(k, k), STRIP(k, k), VX(k), sm); break;
    case 5: larfb_item(cx, VX(k), STRIP(k, k), T(k, j), sub, sm); break;
    case 6: tsqrt_item(cx, T(k, k), T(i, k), STRIP(i, k), sm); break;
    case 7: ssrfb_item(cx, T(i, k), STRIP(i, k), T(k, j), T(i, j), sub, sm); break;
    case 8: {
      const int f = getrf_item(cx, T(k, k), PIV(k, k), VX(k), sm);
      if (f >= 0 && threadIdx.x == 0) atomicMin(cx.info, k * P.b + f + 1);
    } break;
    case 9: gessm_item(cx, VX(k), PIV(k, k), T(k, j), sub, sm); break;
    case 10: {
      const int f = tstrf_item(cx, T(k, k), T(i, k), STRIP(i, k), PIV(i, k), sm);
      if (f >= 0 && threadIdx.x == 0) atomicMin(cx.info, k * P.b + f + 1);
    } break;
    case 11: ssssm_item(cx, T(i, k), STRIP(i, k), PIV(i, k), T(k, j), T(i, j), sub, sm); break;
    default: break;
  }
}

__global__ void __launch_bounds__(TF_THREADS, 1) tf_persistent(Prob P, Sched S) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_it;
  Ctx cx;
  cx.b = P.b;
  cx.ib = P.ib;
  cx.scratch = P.scratch + (size_t)blockIdx.x * P.scr_stride;
  cx.info = P.info;
  cx.abort_flag = S.abort_flag;
  pipe_init(sm);
  for (;;) {
    if (threadIdx.x == 0) s_it = sched_pop(S);
    __syncthreads();
    const int it = s_it;
    if (it < 0) break;
    const int t = S.item_task[it];
    const TaskD d = S.tasks[t];
    const long long t0 = S.trace ? globaltimer() : 0;
    run_item(P, d, it - d.item0, cx, sm);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (S.trace && it < S.trace_cap) {
        long long* r = S.trace + (size_t)it * 5;
        r[0] = t;
        r[1] = it - d.item0;
        r[2] = smid();
        r[3] = t0;
        r[4] = globaltimer();
      }
      sched_complete(S, it);
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(S.exit_count, 1) == (int)gridDim.x - 1) {
      if (ld_volatile(P.info) == INT_MAX) *P.info = 0;
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

// Per-kernel test launcher: one CTA per work item of a single task.
__global__ void __launch_bounds__(TF_THREADS, 1)
    tk_kernel(int kind, int b, int ib, double* t0, double* t1, double* t2, double* aux, int* ipiv, double* vx,
              double* scratch, size_t scr_stride, int* info) {
  extern __shared__ __align__(16) double sm[];
  Ctx cx;
  cx.b = b;
  cx.ib = ib;
  cx.scratch = scratch + (size_t)blockIdx.x * scr_stride;
  cx.info = info;
  cx.abort_flag = nullptr;
  pipe_init(sm);
  const int sub = blockIdx.x;
  int f = -1;
  switch (kind) {
    case 0: f = potrf_item(cx, t0, sm); break;
    case 1: trsm_item(cx, t0, t1, sub, sm); break;
    case 2: syrk_item(cx, t0, t1, sub, sm); break;
    case 3: gemm_item(cx, t0, t1, t2, sub, sm); break;
    case 4: geqrt_item(cx, t0, aux, vx, sm); break;
    case 5: larfb_item(cx, vx, aux, t1, sub, sm); break;
    case 6: tsqrt_item(cx, t0, t1, aux, sm); break;
    case 7: ssrfb_item(cx, t0, aux, t1, t2, sub, sm); break;
    case 8: f = getrf_item(cx, t0, ipiv, vx, sm); break;
    case 9: gessm_item(cx, vx, ipiv, t1, sub, sm); break;
    case 10: f = tstrf_item(cx, t0, t1, aux, ipiv, sm); break;
    case 11: ssssm_item(cx, t0, aux, ipiv, t1, t2, sub, sm); break;
  }
  if (info && threadIdx.x == 0 && blockIdx.x == 0) *info = (f >= 0) ? f + 1 : 0;
}

// unit-lower explicit copy (V_kk / L_kk) of a factored diagonal tile, for tk_run
__global__ void unit_lower_kernel(const double* A, double* X, int b) {
  const size_t bb = (size_t)b * b;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < bb; e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % b), c = (int)(e / b);
    X[e] = (r > c) ? A[e] : (r == c ? 1.0 : 0.0);
  }
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

}  // namespace tf

// ====================================================================================
// Host side
// ====================================================================================
using namespace tf;

namespace {

thread_local char g_err[512] = "";
void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

#define TF_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t _e = (x);                                                               \
    if (_e != cudaSuccess) {                                                            \
      set_err("%s: %s (%s:%d)", #x, cudaGetErrorString(_e), __FILE__, __LINE__);        \
      return TF_ERR_CUDA;                                                               \
    }                                                                                   \
  } while (0)

int g_policy = 1;
int64_t g_trace_cap = 0;
int g_ctas = 0;
std::mutex g_mu;

// ------------------------------------------------------------------ task graph
struct HostDag {
  int alg = 0, p = 0, b = 0, policy = 0;
  std::vector<TaskD> tasks;
  std::vector<int> succ_off, succ, indeg0, item_task, roots;
  int nitems = 0;
  int qbase[NLEV + 1] = {0};
};

inline uint64_t key4(int kind, int k, int i, int j) {
  return ((uint64_t)kind << 60) | ((uint64_t)(unsigned)k << 40) | ((uint64_t)(unsigned)i << 20) | (uint64_t)(unsigned)j;
}

int level_of(int kind, int k, int j, int policy) {
  switch (kind) {
    case 0: case 4: case 8: return 0;      // panel
    case 1: case 6: case 10: return 1;     // couple-factor (TRSM for Cholesky)
    case 5: case 9: return 2;              // row-update
    default:                               // couple-update (SYRK/GEMM/SSRFB/SSSSM)
      return (policy == 1 && j == k + 1) ? 2 : 3;
  }
}

// Build tasks in program order (Algorithms 1-3) and edges by the a13 rules.
void build_dag(HostDag& G, int alg, int p, int b, int policy) {
  G.alg = alg; G.p = p; G.b = b; G.policy = policy;
  std::unordered_map<uint64_t, int> id;
  id.reserve((size_t)p * p * p / 2 + 16);
  auto add = [&](int kind, int k, int i, int j) {
    TaskD d{kind, k, i, j, items_of(kind, b), 0, level_of(kind, k, j, policy), 0};
    id[key4(kind, k, i, j)] = (int)G.tasks.size();
    G.tasks.push_back(d);
  };
  if (alg == 0) {
    for (int k = 0; k < p; ++k) {
      add(0, k, k, k);
      for (int i = k + 1; i < p; ++i) add(1, k, i, k);
      for (int i = k + 1; i < p; ++i)
        for (int j = k + 1; j <= i; ++j) add(i == j ? 2 : 3, k, i, j);
    }
  } else {
    const int F = alg == 1 ? 4 : 8, R = F + 1, C = F + 2, U = F + 3;
    for (int k = 0; k < p; ++k) {
      add(F, k, k, k);
      for (int j = k + 1; j < p; ++j) add(R, k, k, j);
      for (int i = k + 1; i < p; ++i) {
        add(C, k, i, k);
        for (int j = k + 1; j < p; ++j) add(U, k, i, j);
      }
    }
  }
  const int nt = (int)G.tasks.size();
  std::vector<std::vector<int>> preds(nt);
  auto get = [&](int kind, int k, int i, int j) -> int {
    auto it = id.find(key4(kind, k, i, j));
    return it == id.end() ? -1 : it->second;
  };
  for (int t = 0; t < nt; ++t) {
    const TaskD& d = G.tasks[t];
    auto& pr = preds[t];
    auto P = [&](int x) { if (x >= 0) pr.push_back(x); };
    const int k = d.k, i = d.i, j = d.j;
    if (alg == 0) {
      switch (d.kind) {
        case 0: if (k > 0) P(get(2, k - 1, k, k)); break;
        case 1: P(get(0, k, k, k)); if (k > 0) P(get(3, k - 1, i, k)); break;
        case 2: P(get(1, k, i, k)); if (k > 0) P(get(2, k - 1, i, i)); break;
        case 3: P(get(1, k, i, k)); P(get(1, k, j, k)); if (k > 0) P(get(3, k - 1, i, j)); break;
      }
    } else {
      const int F = alg == 1 ? 4 : 8, R = F + 1, C = F + 2, U = F + 3;
      if (d.kind == F) {
        if (k > 0) P(get(U, k - 1, k, k));
      } else if (d.kind == R) {
        P(get(F, k, k, k));
        if (k > 0) P(get(U, k - 1, k, j));
      } else if (d.kind == C) {
        P(i == k + 1 ? get(F, k, k, k) : get(C, k, i - 1, k));
        if (k > 0) P(get(U, k - 1, i, k));
      } else {
        P(get(C, k, i, k));
        P(i == k + 1 ? get(R, k, k, j) : get(U, k, i - 1, j));
        if (k > 0) P(get(U, k - 1, i, j));
      }
    }
  }
  G.indeg0.assign(nt, 0);
  std::vector<int> cnt(nt + 1, 0);
  for (int t = 0; t < nt; ++t) {
    G.indeg0[t] = (int)preds[t].size();
    for (int x : preds[t]) cnt[x + 1]++;
  }
  G.succ_off.assign(nt + 1, 0);
  for (int t = 0; t < nt; ++t) G.succ_off[t + 1] = G.succ_off[t] + cnt[t + 1];
  G.succ.assign(G.succ_off[nt], 0);
  std::vector<int> fill(G.succ_off.begin(), G.succ_off.end() - 1);
  for (int t = 0; t < nt; ++t)
    for (int x : preds[t]) G.succ[fill[x]++] = t;
  // items and per-level queue capacity
  int lev_items[NLEV] = {0};
  G.nitems = 0;
  for (int t = 0; t < nt; ++t) {
    G.tasks[t].item0 = G.nitems;
    G.nitems += G.tasks[t].nitems;
    lev_items[G.tasks[t].level] += G.tasks[t].nitems;
  }
  G.item_task.resize(G.nitems);
  for (int t = 0; t < nt; ++t)
    for (int x = 0; x < G.tasks[t].nitems; ++x) G.item_task[G.tasks[t].item0 + x] = t;
  G.qbase[0] = 0;
  for (int l = 0; l < NLEV; ++l) G.qbase[l + 1] = G.qbase[l] + lev_items[l];
  G.roots.clear();
  for (int t = 0; t < nt; ++t)
    if (G.indeg0[t] == 0) G.roots.push_back(t);
}

struct DevDag {
  std::shared_ptr<HostDag> h;
  TaskD* tasks = nullptr;
  int *succ_off = nullptr, *succ = nullptr, *item_task = nullptr, *indeg0 = nullptr, *roots = nullptr;
};

std::map<std::tuple<int, int, int, int, int>, DevDag> g_dags;  // (dev, alg, p, b, policy)

template <class T>
int upload(T** dst, const std::vector<T>& v) {
  TF_CUDA(cudaMalloc(dst, sizeof(T) * (v.empty() ? 1 : v.size())));
  if (!v.empty()) TF_CUDA(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return 0;
}

int get_dag(int dev, int alg, int p, int b, DevDag** out) {
  auto key = std::make_tuple(dev, alg, p, b, g_policy);
  auto it = g_dags.find(key);
  if (it != g_dags.end()) { *out = &it->second; return 0; }
  DevDag D;
  D.h = std::make_shared<HostDag>();
  build_dag(*D.h, alg, p, b, g_policy);
  int rc;
  if ((rc = upload(&D.tasks, D.h->tasks))) return rc;
  if ((rc = upload(&D.succ_off, D.h->succ_off))) return rc;
  if ((rc = upload(&D.succ, D.h->succ))) return rc;
  if ((rc = upload(&D.item_task, D.h->item_task))) return rc;
  if ((rc = upload(&D.indeg0, D.h->indeg0))) return rc;
  if ((rc = upload(&D.roots, D.h->roots))) return rc;
  auto res = g_dags.emplace(key, D);
  *out = &res.first->second;
  return 0;
}

// ------------------------------------------------------------------ workspaces
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};
int ensure(Buf& b, size_t bytes) {
  if (b.bytes >= bytes && b.p) return 0;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
    cudaGetLastError();
    set_err("cudaMalloc(%zu) failed", bytes);
    return TF_ERR_NOMEM;
  }
  b.bytes = bytes;
  return 0;
}

struct Workspace {
  Buf state, q, vx, scratch, info, trace;
  Buf hostA, hostAux, hostPiv;  // device buffers for tile_factor_host
  int64_t last_items = 0;
  cudaStream_t stream = nullptr;
};
std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;

int g_nsm[64] = {0};
bool g_attr_set[64] = {false};
Workspace* g_last_ws = nullptr;

size_t smem_bytes() { return (size_t)SMEM_DOUBLES * sizeof(double); }

int device_setup(int dev) {
  if (dev >= 64) { set_err("device id %d too large", dev); return TF_ERR_UNSUPPORTED; }
  if (!g_attr_set[dev]) {
    TF_CUDA(cudaDeviceGetAttribute(&g_nsm[dev], cudaDevAttrMultiProcessorCount, dev));
    TF_CUDA(cudaFuncSetAttribute(tf_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
    TF_CUDA(cudaFuncSetAttribute(tk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
    g_attr_set[dev] = true;
  }
  return 0;
}

size_t scr_stride_for(int b, int ib) { return ((size_t)2 * ib * b + 64 + 31) & ~(size_t)31; }

int check_args(int64_t n, int64_t b, int64_t ib, const void* dA) {
  if (n <= 0) { set_err("n must be > 0"); return -1; }
  if (b <= 0 || n % b) { set_err("b must be > 0 and divide n"); return -2; }
  if (b > TF_MAX_B) { set_err("b > TF_MAX_B"); return -2; }
  if (ib <= 0 || b % ib) { set_err("ib must be > 0 and divide b"); return -3; }
  if (!dA) { set_err("null matrix pointer"); return -4; }
  if ((n / b) > (1 << 19)) { set_err("too many tiles"); return -1; }
  return 0;
}

int run_factorization(int alg, int64_t n, int64_t b, int64_t ib, double* dA, double* aux, int32_t* ipiv,
                      int32_t* d_info, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  int rc;
  if ((rc = device_setup(dev))) return rc;
  const int p = (int)(n / b);
  DevDag* D;
  if ((rc = get_dag(dev, alg, p, (int)b, &D))) return rc;
  const HostDag& H = *D->h;
  Workspace& W = g_ws[std::make_pair(dev, stream)];
  W.stream = stream;
  const int nt = (int)H.tasks.size();
  const int ctas = g_ctas > 0 ? g_ctas : g_nsm[dev];
  const size_t state_ints = (size_t)2 * nt + 2 * NLEV + 8;
  if ((rc = ensure(W.state, state_ints * sizeof(int)))) return rc;
  if ((rc = ensure(W.q, (size_t)H.nitems * sizeof(int)))) return rc;
  if (alg != 0 && (rc = ensure(W.vx, (size_t)p * b * b * sizeof(double)))) return rc;
  const size_t scr = scr_stride_for((int)b, (int)ib);
  if ((rc = ensure(W.scratch, scr * ctas * sizeof(double)))) return rc;
  if ((rc = ensure(W.info, 64))) return rc;
  if (g_trace_cap > 0 && (rc = ensure(W.trace, (size_t)H.nitems * 5 * sizeof(long long)))) return rc;
  int* st = (int*)W.state.p;
  Sched S;
  S.tasks = D->tasks;
  S.succ_off = D->succ_off;
  S.succ = D->succ;
  S.item_task = D->item_task;
  S.ntasks = nt;
  S.nitems = H.nitems;
  for (int l = 0; l <= NLEV; ++l) S.qbase[l] = H.qbase[l];
  S.indeg = st;
  S.items_done = st + nt;
  S.head = st + 2 * nt;
  S.tail = S.head + NLEV;
  S.ndone = S.tail + NLEV;
  S.abort_flag = S.ndone + 1;
  S.exit_count = S.ndone + 2;
  S.q = (int*)W.q.p;
  S.trace = g_trace_cap > 0 ? (long long*)W.trace.p : nullptr;
  S.trace_cap = g_trace_cap > 0 ? H.nitems : 0;
  W.last_items = g_trace_cap > 0 ? H.nitems : 0;
  Prob P;
  P.A = dA;
  P.aux = aux;
  P.ipiv = ipiv;
  P.vx = (double*)W.vx.p;
  P.scratch = (double*)W.scratch.p;
  P.scr_stride = scr;
  P.n = (int)n;
  P.b = (int)b;
  P.ib = (int)ib;
  P.p = p;
  P.info = d_info ? d_info : (int*)W.info.p;
  tf_sched_reset<<<64, 256, 0, stream>>>(S, D->indeg0, H.nitems, P.info);
  tf_sched_seed<<<1, 32, 0, stream>>>(S, D->roots, (int)H.roots.size());
  tf_persistent<<<ctas, TF_THREADS, smem_bytes(), stream>>>(P, S);
  TF_CUDA(cudaGetLastError());
  g_last_ws = &W;
  return 0;
}

}  // namespace

// ====================================================================================
// C-ABI
// ====================================================================================
extern "C" {

int tile_chol(int64_t n, int64_t b, int64_t ib, double* dA, int32_t* d_info, tf_stream_t stream) {
  int rc = check_args(n, b, ib, dA);
  if (rc) return rc;
  return run_factorization(0, n, b, ib, dA, nullptr, nullptr, d_info, (cudaStream_t)stream);
}

int tile_qr(int64_t n, int64_t b, int64_t ib, double* dA, double* dT, tf_stream_t stream) {
  int rc = check_args(n, b, ib, dA);
  if (rc) return rc;
  if (!dT) { set_err("null T pointer"); return -5; }
  return run_factorization(1, n, b, ib, dA, dT, nullptr, nullptr, (cudaStream_t)stream);
}

int tile_lu(int64_t n, int64_t b, int64_t ib, double* dA, double* dLs, int32_t* dIpiv, int32_t* d_info,
            tf_stream_t stream) {
  int rc = check_args(n, b, ib, dA);
  if (rc) return rc;
  if (!dLs) { set_err("null L-strip pointer"); return -5; }
  if (!dIpiv) { set_err("null ipiv pointer"); return -6; }
  return run_factorization(2, n, b, ib, dA, dLs, dIpiv, d_info, (cudaStream_t)stream);
}

size_t tile_qr_t_elems(int64_t n, int64_t b, int64_t ib) {
  if (n <= 0 || b <= 0 || n % b) return 0;
  const size_t p = n / b;
  return p * p * (size_t)ib * b;
}
size_t tile_lu_l_elems(int64_t n, int64_t b, int64_t ib) { return tile_qr_t_elems(n, b, ib); }
size_t tile_lu_ipiv_elems(int64_t n, int64_t b) {
  if (n <= 0 || b <= 0 || n % b) return 0;
  const size_t p = n / b;
  return p * p * (size_t)b;
}

int tile_pack(int64_t m, int64_t n, int64_t b, const double* dDense, double* dTiles, tf_stream_t stream) {
  if (m <= 0 || n <= 0) return -1;
  if (b <= 0 || m % b || n % b) return -3;
  if (!dDense) return -4;
  if (!dTiles) return -5;
  pack_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(m, n, b, const_cast<double*>(dDense), dTiles, 0);
  TF_CUDA(cudaGetLastError());
  return 0;
}

int tile_unpack(int64_t m, int64_t n, int64_t b, const double* dTiles, double* dDense, tf_stream_t stream) {
  if (m <= 0 || n <= 0) return -1;
  if (b <= 0 || m % b || n % b) return -3;
  if (!dTiles) return -4;
  if (!dDense) return -5;
  pack_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(m, n, b, dDense, const_cast<double*>(dTiles), 1);
  TF_CUDA(cudaGetLastError());
  return 0;
}

int tile_factor_host(int kind, int64_t n, int64_t b, int64_t ib, double* hA, double* hAux, int32_t* hIpiv,
                     int32_t* hInfo, tf_stream_t stream) {
  int rc = check_args(n, b, ib, hA);
  if (rc) return rc;
  if (kind < 0 || kind > 2) return -1;
  cudaStream_t s = (cudaStream_t)stream;
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  Workspace* W;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    W = &g_ws[std::make_pair(dev, s)];
  }
  const size_t an = (size_t)n * n;
  const size_t xn = kind == 0 ? 0 : tile_qr_t_elems(n, b, ib);
  const size_t pn = kind == 2 ? tile_lu_ipiv_elems(n, b) : 0;
  if ((rc = ensure(W->hostA, an * sizeof(double) + 64))) return rc;
  if (xn && (rc = ensure(W->hostAux, xn * sizeof(double)))) return rc;
  if (pn && (rc = ensure(W->hostPiv, pn * sizeof(int32_t) + 64))) return rc;
  double* dA = (double*)W->hostA.p;
  int32_t* dInfo = (int32_t*)((char*)W->hostA.p + an * sizeof(double));
  TF_CUDA(cudaMemcpyAsync(dA, hA, an * sizeof(double), cudaMemcpyHostToDevice, s));
  if (kind == 0) rc = tile_chol(n, b, ib, dA, dInfo, stream);
  else if (kind == 1) rc = tile_qr(n, b, ib, dA, (double*)W->hostAux.p, stream);
  else rc = tile_lu(n, b, ib, dA, (double*)W->hostAux.p, (int32_t*)W->hostPiv.p, dInfo, stream);
  if (rc) return rc;
  TF_CUDA(cudaMemcpyAsync(hA, dA, an * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (hAux && xn) TF_CUDA(cudaMemcpyAsync(hAux, W->hostAux.p, xn * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (hIpiv && pn) TF_CUDA(cudaMemcpyAsync(hIpiv, W->hostPiv.p, pn * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  if (hInfo) {
    if (kind == 1) *hInfo = 0;
    else TF_CUDA(cudaMemcpyAsync(hInfo, dInfo, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  }
  TF_CUDA(cudaStreamSynchronize(s));
  return 0;
}

void tile_set_policy(int policy) { g_policy = (policy == 0) ? 0 : 1; }
void tile_set_trace(int64_t cap) { g_trace_cap = cap > 0 ? cap : 0; }
void tile_set_ctas(int ctas) { g_ctas = ctas > 0 ? ctas : 0; }

int64_t tile_trace_fetch(int64_t* rec, int64_t cap) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_last_ws || !g_last_ws->trace.p || g_last_ws->last_items == 0) return 0;
  if (cudaStreamSynchronize(g_last_ws->stream) != cudaSuccess) return -1;
  int64_t nrec = g_last_ws->last_items;
  if (cap < nrec) nrec = cap;
  if (rec && nrec > 0 &&
      cudaMemcpy(rec, g_last_ws->trace.p, (size_t)nrec * 5 * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return nrec;
}

int64_t tile_dag_export(int alg, int64_t p, int policy, int32_t* kind, int32_t* k, int32_t* i, int32_t* j,
                        int32_t* level, int64_t cap, int64_t* succ_off, int32_t* succ, int64_t succ_cap,
                        int64_t* nedges) {
  if (alg < 0 || alg > 2 || p <= 0) return -1;
  HostDag G;
  build_dag(G, alg, (int)p, 128, policy);
  const int64_t nt = (int64_t)G.tasks.size();
  for (int64_t t = 0; t < nt && t < cap; ++t) {
    if (kind) kind[t] = G.tasks[t].kind;
    if (k) k[t] = G.tasks[t].k;
    if (i) i[t] = G.tasks[t].i;
    if (j) j[t] = G.tasks[t].j;
    if (level) level[t] = G.tasks[t].level;
  }
  if (succ_off && cap >= nt)
    for (int64_t t = 0; t <= nt; ++t) succ_off[t] = G.succ_off[t];
  const int64_t ne = (int64_t)G.succ.size();
  if (succ)
    for (int64_t e = 0; e < ne && e < succ_cap; ++e) succ[e] = G.succ[e];
  if (nedges) *nedges = ne;
  return nt;
}

int tk_run(int kind, int64_t b, int64_t ib, double* t0, double* t1, double* t2, double* aux, int32_t* ipiv,
           int32_t* d_info, tf_stream_t stream) {
  if (kind < 0 || kind > 11) return -1;
  if (b <= 0 || b > TF_MAX_B) return -2;
  if (ib <= 0 || b % ib) return -3;
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(g_mu);
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  int rc;
  if ((rc = device_setup(dev))) return rc;
  Workspace& W = g_ws[std::make_pair(dev, s)];
  const int items = items_of(kind, (int)b);
  const size_t scr = scr_stride_for((int)b, (int)ib);
  if ((rc = ensure(W.scratch, scr * items * sizeof(double)))) return rc;
  if ((rc = ensure(W.vx, (size_t)b * b * sizeof(double)))) return rc;
  double* vx = (double*)W.vx.p;
  if (kind == 5 || kind == 9) {
    unit_lower_kernel<<<64, 256, 0, s>>>(t0, vx, (int)b);
    TF_CUDA(cudaGetLastError());
  }
  tk_kernel<<<items, TF_THREADS, smem_bytes(), s>>>(kind, (int)b, (int)ib, t0, t1, t2, aux, ipiv, vx,
                                                     (double*)W.scratch.p, scr, d_info);
  TF_CUDA(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------- multi-GPU (see tf_dist.cpp)

const char* tile_strerror(int code) {
  switch (code) {
    case 0: return "success";
    case TF_ERR_CUDA: return "CUDA runtime error";
    case TF_ERR_NOMEM: return "device allocation failed";
    case TF_ERR_NCCL: return "NCCL error";
    case TF_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return code < 0 ? "invalid argument" : "unknown error";
  }
}

const char* tile_last_error(void) { return g_err; }

void tile_finalize(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& kv : g_ws) {
    Workspace& W = kv.second;
    for (Buf* b : {&W.state, &W.q, &W.vx, &W.scratch, &W.info, &W.trace, &W.hostA, &W.hostAux, &W.hostPiv})
      if (b->p) cudaFree(b->p);
  }
  g_ws.clear();
  for (auto& kv : g_dags) {
    DevDag& D = kv.second;
    cudaFree(D.tasks);
    cudaFree(D.succ_off);
    cudaFree(D.succ);
    cudaFree(D.item_task);
    cudaFree(D.indeg0);
    cudaFree(D.roots);
  }
  g_dags.clear();
  g_last_ws = nullptr;
  for (int d = 0; d < 64; ++d) g_attr_set[d] = false;
}

}  // extern "C"
