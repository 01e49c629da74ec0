// tf_host.cpp — host side of libtilefact.so: the task-graph builder (Algorithms 1-3 with
// the SURVEY §8(a) a13 dependency rules), the multi-GPU distribution plan, workspace
// caches, and the C-ABI declared in include/tilefact.h.  No device code lives here; the
// kernels and their launch wrappers are in tf_device.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/tilefact.h"
#include "tf_sched.h"

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

#define TF_LAUNCH(x)                                                                    \
  do {                                                                                  \
    int _e = (x);                                                                       \
    if (_e) {                                                                           \
      set_err("%s: %s", #x, cudaGetErrorString((cudaError_t)_e));                       \
      return TF_ERR_CUDA;                                                               \
    }                                                                                   \
  } while (0)

int g_policy = 1;
int g_slab_dag = -1;  // tile_set_slab_dag: -1 = default (TF_FINE env, on), 0 = tile-level, 1 = slab-level
int64_t g_trace_cap = 0;
int g_ctas = 0;
std::recursive_mutex g_mu;

// ------------------------------------------------------------------ task graph
struct HostDag {
  int alg = 0, p = 0, b = 0, policy = 0;
  std::vector<TaskD> tasks;
  std::vector<int> succ_off, succ, indeg0, item_task, roots;
  std::vector<SendEnt> sends;
  int nitems = 0;
  int qbase[NLEV + 1] = {0};
};

inline uint64_t key4(int kind, int k, int i, int j) {
  return ((uint64_t)kind << 60) | ((uint64_t)(unsigned)k << 40) | ((uint64_t)(unsigned)i << 20) | (uint64_t)(unsigned)j;
}

int level_of(int kind, int k, int j, int policy) {
  switch (kind) {
    case K_UNITL: case K_XTRSMU: case K_XGESSM: case K_XLARFB: case K_XUNGESSM: return 1;
    case K_XSSSSM: case K_XSSRFB: case K_XUNSSSSM: return 2;
    case K_XGEMM: return 3;
    case 0: case 4: case 8: case K_SEND: case K_RECV: return 0;  // panel (and panel traffic)
    case 1: case 6: case 10: return 1;     // couple-factor (TRSM for Cholesky)
    case 5: case 9: return 2;              // row-update
    default:                               // couple-update (SYRK/GEMM/SSRFB/SSSSM)
      return (policy == 1 && j == k + 1) ? 2 : 3;
  }
}

// Tasks of Algorithms 1-3 in program order and their predecessor lists (a13 rules).
// qc: tile columns (QR / LU on a p x qc tiled matrix; k < min(p, qc));
// < 0 = square.
void global_tasks(int alg, int p, int b, int ib, int policy, std::vector<TaskD>& tasks,
                  std::vector<std::vector<int>>& preds, int qc = -1) {
  if (qc < 0) qc = p;
  std::unordered_map<uint64_t, int> id;
  id.reserve((size_t)p * p * p / 2 + 16);
  tasks.clear();
  auto add = [&](int kind, int k, int i, int j) {
    TaskD d{kind, k, i, j, items_of(kind, b, ib), 0, level_of(kind, k, j, policy), 0};
    id[key4(kind, k, i, j)] = (int)tasks.size();
    tasks.push_back(d);
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
    const int kk = p < qc ? p : qc;
    for (int k = 0; k < kk; ++k) {
      add(F, k, k, k);
      for (int j = k + 1; j < qc; ++j) add(R, k, k, j);
      for (int i = k + 1; i < p; ++i) {
        add(C, k, i, k);
        for (int j = k + 1; j < qc; ++j) add(U, k, i, j);
      }
    }
  }
  const int nt = (int)tasks.size();
  preds.assign(nt, {});
  auto get = [&](int kind, int k, int i, int j) -> int {
    auto it = id.find(key4(kind, k, i, j));
    return it == id.end() ? -1 : it->second;
  };
  for (int t = 0; t < nt; ++t) {
    const TaskD& d = tasks[t];
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
}

// Slab-level DAG of Algorithms 2-3 (QR / LU on the register-slab kernels, single GPU).
// The panel tasks become one task per 32-column slab s (GEQRT / GETRF: FS(k,s); TSQRT /
// TSTRF: CS(k,i,s)), and the update tasks of the next panel column, LARFB / GESSM (k,k+1)
// and SSRFB / SSSSM (k,i,k+1), one task per slab item.  Every slab of a panel task reads
// only global results of the slabs before it (left-looking) and touches the diagonal tile
// only in its own columns (TSQRT / TSTRF: the upper part of R_kk / U_kk; GETRF's later
// interchanges move only rows below the slab's diagonal block), so
//   FS(k,s)      <- FS(k,s-1), U(k-1,k,k) slab s
//   CS(k,i,s)    <- CS(k,i,s-1), [i == k+1 ? FS(k,s) : CS(k,i-1,s)], U(k-1,i,k) slab s
//   R(k,j)[s]    <- FS(k,last), U(k-1,k,j)
//   U(k,i,j)[s]  <- CS(k,i,last), [i == k+1 ? R(k,j)[s] : U(k,i-1,j)[s]], U(k-1,i,j)
// (slab s where the producer is split, the whole task otherwise).  Consecutive TSQRT /
// TSTRF of a tile column then overlap slab by slab, and the next panel starts on its
// first slab while the lookahead updates of its later slabs run; each tile sees the same
// operations in the same order as in the tile-level DAG (results are bitwise identical).
void global_tasks_fine(int alg, int p, int b, int ib, int policy, std::vector<TaskD>& tasks,
                       std::vector<std::vector<int>>& preds, int qc = -1) {
  if (qc < 0) qc = p;
  const int S = b / NSR;
  const int F = alg == 1 ? 4 : 8, R = F + 1, C = F + 2, U = F + 3;
  const int FS = alg == 1 ? K_GEQRT_S : K_GETRF_S, CS = alg == 1 ? K_TSQRT_S : K_TSTRF_S;
  const int CA = alg == 1 ? K_TSQRT_A : K_TSTRF_A;
  // finished inner blocks before slab s; the last slab of inner block t
  auto nfull = [&](int s) { return (s * NSR - (s * NSR) % ib) / ib; };
  auto last_slab = [&](int t) { return (t + 1) * ib / NSR - 1; };
  std::unordered_map<uint64_t, int> id;
  tasks.clear();
  // split (per-slab) tasks: key kind | 32, j' = j * 64 + s
  auto key = [&](int kind, int k, int i, int j, int s) {
    return s < 0 ? key4(kind, k, i, j) : key4(kind | 32, k, i, j * 64 + s);
  };
  auto add = [&](int kind, int k, int i, int j, int s, int nit) {
    TaskD d{kind, k, i, j, nit, 0, level_of(coarse_kind(kind), k, j, policy), s < 0 ? 0 : s};
    id[key(kind, k, i, j, s)] = (int)tasks.size();
    tasks.push_back(d);
  };
  const int nit = items_of(U, b, ib);  // slab items of an update task (= S)
  const int kk = p < qc ? p : qc;
  for (int k = 0; k < kk; ++k) {
    for (int s = 0; s < S; ++s) add(FS, k, k, k, s, 1);
    for (int j = k + 1; j < qc; ++j) {
      if (j == k + 1) for (int s = 0; s < nit; ++s) add(R, k, k, j, s, 1);
      else add(R, k, k, j, -1, nit);
    }
    for (int i = k + 1; i < p; ++i) {
      for (int s = 0; s < S; ++s) {
        if (ts_apply_split(alg == 2) && nfull(s) >= 2) add(CA, k, i, k, s, 1);  // older inner blocks, off the chain
        add(CS, k, i, k, s, 1);
      }
      for (int j = k + 1; j < qc; ++j) {
        if (j == k + 1) for (int s = 0; s < nit; ++s) add(U, k, i, j, s, 1);
        else add(U, k, i, j, -1, nit);
      }
    }
  }
  auto get = [&](int kind, int k, int i, int j, int s) -> int {
    auto it = id.find(key(kind, k, i, j, s));
    return it == id.end() ? -1 : it->second;
  };
  // update task (k,i,j) or its slab s (split iff j == k + 1); s = -1: the whole task
  auto upd = [&](int kind, int k, int i, int j, int s) { return get(kind, k, i, j, j == k + 1 ? s : -1); };
  const int nt = (int)tasks.size();
  preds.assign(nt, {});
  for (int t = 0; t < nt; ++t) {
    const TaskD& d = tasks[t];
    auto& pr = preds[t];
    auto P = [&](int x) { if (x >= 0 && std::find(pr.begin(), pr.end(), x) == pr.end()) pr.push_back(x); };
    const int k = d.k, i = d.i, j = d.j, s = d.pad;
    const bool split = d.nitems == 1 && (d.kind == R || d.kind == U);
    if (d.kind == FS) {
      if (s > 0) P(get(FS, k, k, k, s - 1));
      if (k > 0) P(upd(U, k - 1, k, k, s));
    } else if (d.kind == CA) {
      // inner blocks [0, nfull(s) - 1) of TSQRT / TSTRF (i,k) applied to slab s: after block
      // nfull(s) - 2 is factored, the previous TSQRT / TSTRF of the column left slab s of the
      // diagonal tile, and step k-1 updated slab s of tile (i,k)
      P(get(CS, k, i, k, last_slab(nfull(s) - 2)));
      P(i == k + 1 ? get(FS, k, k, k, s) : get(CS, k, i - 1, k, s));
      if (k > 0) P(upd(U, k - 1, i, k, s));
    } else if (d.kind == CS) {
      if (s > 0) P(get(CS, k, i, k, s - 1));
      const int ca = get(CA, k, i, k, s);
      if (ca >= 0) {
        P(ca);
      } else {
        P(i == k + 1 ? get(FS, k, k, k, s) : get(CS, k, i - 1, k, s));
        if (k > 0) P(upd(U, k - 1, i, k, s));
      }
    } else if (d.kind == R) {
      P(get(FS, k, k, k, S - 1));
      if (k > 0) P(upd(U, k - 1, k, j, split ? s : -1));
    } else if (d.kind == U) {
      P(get(CS, k, i, k, S - 1));
      const int sx = split ? s : -1;  // (j == k + 1 exactly when split)
      P(i == k + 1 ? get(R, k, k, j, sx) : get(U, k, i - 1, j, sx));
      if (k > 0) P(get(U, k - 1, i, j, -1));  // split iff j == k; here j >= k + 1: the whole task
    }
  }
}

// Panel-level DAG of Algorithm 1 (Cholesky, b a multiple of 128 and >= 256, single GPU).
// POTRF(k) and TRSM(k,i) are left-looking over nr = b / 128 column panels (potrf_blocked,
// trsm_right): panel J of a row block needs the panels to its left of that row block and of
// block row J, and the factored diagonal block (J,J).  As tasks:
//   PD(k,J)   diagonal block of panel J   <- PB(k,J-1)  [J = 0: SYRK(k-1,k,k)]
//   PB(k,J)   blocks below it (nr-1-J items) <- PD(k,J)
//   TP(k,i,J) panel J of TRSM(k,i) (nr items)  <- PD(k,J), TP(k,i,J-1)  [J = 0: GEMM(k-1,i,k)]
//   SYRK(k,i,i) / GEMM(k,i,j) <- TP(k,.,nr-1) as before
// (PD(k,J) <- PB(k,J-1) <- PD(k,J-1) ... orders every earlier panel of the diagonal tile
// before it.)  The per-step chain POTRF -> TRSM shrinks from the whole POTRF plus a whole
// TRSM to 2 nr - 1 block kernels plus one TRSM panel; every element sees the same
// operations in the same order as in the tile-level DAG (results are bitwise identical).
// Optional (tile_set_gemm_tile_min / TF_GEMM_TILE_MIN = t > 0; default off): GEMM(k,i,j)
// outside the lookahead column runs as ONE whole-tile item (pad = 1, gemm_tile_body: the
// nr x nr sub-tile products as one slice stream) while step k has at least t such tiles, so
// the per-item costs (scheduler round trip, pipeline fill, last epilogue) are paid once per
// tile; later steps and the lookahead column keep the finer strip items.  Measured on
// config 4 with t = 296: 386.4 -> 385.4 ms but DRAM traffic 344 -> 430 GB per launch (the four
// strip items of a tile run on neighbouring CTAs at the same time and share B through L2;
// whole-tile items each stream their own 6 MB): not worth it, so it is off by default.
int g_gemm_tile_min = -1;  // tile_set_gemm_tile_min: -1 = default (TF_GEMM_TILE_MIN env, else 0 = off)
int gemm_tile_min() {
  static const int env = getenv("TF_GEMM_TILE_MIN") ? atoi(getenv("TF_GEMM_TILE_MIN")) : 0;
  return g_gemm_tile_min >= 0 ? g_gemm_tile_min : env;
}

void global_tasks_chol_panel(int p, int b, int policy, std::vector<TaskD>& tasks,
                             std::vector<std::vector<int>>& preds) {
  const int nr = b / 128;
  const int tile_min = gemm_tile_min();
  std::unordered_map<uint64_t, int> id;
  id.reserve((size_t)p * p * p / 2 + 16);
  tasks.clear();
  // local kind codes for the key: 0 PD, 1 PB, 2 TP, 3 SYRK, 4 GEMM; panel in the low 6 bits of
  // j (nr <= 32 for b <= TF_MAX_B = 4096)
  auto key = [&](int lk, int k, int i, int j, int J) { return key4(lk, k, i, j * 64 + J); };
  auto add = [&](int lk, int kind, int k, int i, int j, int J, int nit, int pad = -1) {
    TaskD d{kind, k, i, j, nit, 0, level_of(coarse_kind(kind), k, j, policy), pad >= 0 ? pad : J};
    id[key(lk, k, i, j, J)] = (int)tasks.size();
    tasks.push_back(d);
  };
  for (int k = 0; k < p; ++k) {
    for (int J = 0; J < nr; ++J) {
      add(0, K_POTRF_D, k, k, k, J, 1);
      if (J + 1 < nr) add(1, K_POTRF_B, k, k, k, J, nr - 1 - J);
    }
    for (int i = k + 1; i < p; ++i)
      for (int J = 0; J < nr; ++J) add(2, K_TRSM_P, k, i, k, J, nr);
    const int m = p - k - 1;
    const bool whole = tile_min > 0 && (m - 1) * (m - 2) / 2 >= tile_min;  // GEMM tiles with j > k + 1
    for (int i = k + 1; i < p; ++i)
      for (int j = k + 1; j <= i; ++j) {
        if (i == j) add(3, 2, k, i, j, 0, items_of(2, b, 0));
        else if (whole && j > k + 1) add(4, 3, k, i, j, 0, 1, /*pad=*/1);
        else add(4, 3, k, i, j, 0, items_of(3, b, 0));
      }
  }
  auto get = [&](int lk, int k, int i, int j, int J) -> int {
    auto it = id.find(key(lk, k, i, j, J));
    return it == id.end() ? -1 : it->second;
  };
  const int nt = (int)tasks.size();
  preds.assign(nt, {});
  for (int t = 0; t < nt; ++t) {
    const TaskD& d = tasks[t];
    auto& pr = preds[t];
    auto P = [&](int x) { if (x >= 0) pr.push_back(x); };
    const int k = d.k, i = d.i, j = d.j, J = d.pad;
    switch (d.kind) {
      case K_POTRF_D:
        if (J > 0) P(get(1, k, k, k, J - 1));
        else if (k > 0) P(get(3, k - 1, k, k, 0));
        break;
      case K_POTRF_B: P(get(0, k, k, k, J)); break;
      case K_TRSM_P:
        P(get(0, k, k, k, J));
        if (J > 0) P(get(2, k, i, k, J - 1));
        else if (k > 0) P(get(4, k - 1, i, k, 0));
        break;
      case 2: P(get(2, k, i, k, nr - 1)); if (k > 0) P(get(3, k - 1, i, i, 0)); break;
      case 3:
        P(get(2, k, i, k, nr - 1)); P(get(2, k, j, k, nr - 1));
        if (k > 0) P(get(4, k - 1, i, j, 0));
        break;
    }
  }
}

// Solve / apply DAGs (NEXT-3) over the right-hand-side tiles X(i,c), c < q.  The factor
// tiles are read-only inputs, so dependencies come from the X tiles and the explicit
// unit-lower copies VX(k) only; they are derived generically (read-after-write,
// write-after-read, write-after-write on each tile, tasks in program order), which is
// correct by construction for any task order below.
//   getrs: N^{-1} X (XGESSM(k), XSSSSM(i>k,k): Algorithm 3's updates on extra columns),
//          then U^{-1} X (XTRSMU(k), XGEMM(i<k,k), k descending)
//   ormqr: Q^T X (XLARFB(k), XSSRFB(i>k,k): Algorithm 2's updates on extra columns)
//   qrs:   ormqr, then R^{-1} X as getrs' second half
//   lu_apply_N: N X = every elimination step undone in reverse program order (C4)
void solve_tasks(int alg, int p, int b, int ib, int q, int policy, std::vector<TaskD>& tasks,
                 std::vector<std::vector<int>>& preds) {
  struct Acc { int tile; bool w; };
  std::vector<std::vector<Acc>> acc;
  tasks.clear();
  const int VXB = p * q;  // tile ids: X(i,c) = i + c*p, VX(k) = VXB + k
  auto X = [&](int i, int c) { return i + c * p; };
  auto add = [&](int kind, int k, int i, int j, std::vector<Acc> a) {
    tasks.push_back(TaskD{kind, k, i, j, items_of(kind, b, ib), 0, level_of(kind, k, j, policy), 0});
    acc.push_back(std::move(a));
  };
  const bool lu = alg == ALG_GETRS || alg == ALG_LUN;
  if (alg == ALG_GETRS || alg == ALG_ORMQR || alg == ALG_QRS) {
    for (int k = 0; k < p; ++k) add(K_UNITL, k, k, k, {{VXB + k, true}});
    for (int k = 0; k < p; ++k) {
      for (int c = 0; c < q; ++c)
        add(lu ? K_XGESSM : K_XLARFB, k, k, c, {{VXB + k, false}, {X(k, c), true}});
      for (int i = k + 1; i < p; ++i)
        for (int c = 0; c < q; ++c) add(lu ? K_XSSSSM : K_XSSRFB, k, i, c, {{X(k, c), true}, {X(i, c), true}});
    }
  }
  if (alg == ALG_GETRS || alg == ALG_QRS) {
    for (int k = p - 1; k >= 0; --k)
      for (int c = 0; c < q; ++c) {
        add(K_XTRSMU, k, k, c, {{X(k, c), true}});
        for (int i = 0; i < k; ++i) add(K_XGEMM, k, i, c, {{X(k, c), false}, {X(i, c), true}});
      }
  }
  if (alg == ALG_LUN) {
    for (int k = p - 1; k >= 0; --k)
      for (int c = 0; c < q; ++c) {
        for (int i = p - 1; i > k; --i) add(K_XUNSSSSM, k, i, c, {{X(k, c), true}, {X(i, c), true}});
        add(K_XUNGESSM, k, k, c, {{X(k, c), true}});
      }
  }
  const int nt = (int)tasks.size();
  preds.assign(nt, {});
  std::unordered_map<int, int> last_w;
  std::unordered_map<int, std::vector<int>> readers;
  for (int t = 0; t < nt; ++t) {
    auto& pr = preds[t];
    for (const Acc& a : acc[t]) {
      auto lw = last_w.find(a.tile);
      if (lw != last_w.end()) pr.push_back(lw->second);
      if (!a.w) {
        readers[a.tile].push_back(t);
      } else {
        for (int r : readers[a.tile])
          if (r != t) pr.push_back(r);
        readers[a.tile].clear();
        last_w[a.tile] = t;
      }
    }
    std::sort(pr.begin(), pr.end());
    pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
  }
}

// CSR successors, in-degrees, work items, per-level queue bases and roots.
void finalize_dag(HostDag& G, const std::vector<std::vector<int>>& preds) {
  const int nt = (int)G.tasks.size();
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
    if (G.indeg0[t] == 0 && G.tasks[t].kind != K_RECV && G.tasks[t].kind != K_ARRIVE) G.roots.push_back(t);
}

// Host <-> device copy overlap (tile_factor_host): ARRIVE(j) before the first task that
// touches a tile of column j, DONE(j) after the last task that writes one.  Tile sets per
// task as in the a13 rules (reads of the panel tiles, writes of the outputs).
void add_copy_tasks(int alg, int p, int b, int ib, std::vector<TaskD>& tasks, std::vector<std::vector<int>>& preds) {
  const int nt = (int)tasks.size();
  std::vector<char> touched((size_t)p * p, 0);
  std::vector<int> lastw((size_t)p * p, -1);
  auto id = [&](int i, int j) { return (size_t)i + (size_t)j * p; };
  const int a0 = nt;  // ARRIVE(j) = a0 + j, DONE(j) = a0 + p + j
  for (int j = 0; j < p; ++j) tasks.push_back(TaskD{K_ARRIVE, j, j, j, 1, 0, 0, 0});
  for (int j = 0; j < p; ++j) tasks.push_back(TaskD{K_DONE, j, j, j, 1, 0, 0, 0});
  preds.resize(tasks.size());
  for (int t = 0; t < nt; ++t) {
    const TaskD& d = tasks[t];
    const int k = d.k, i = d.i, j = d.j, kind = coarse_kind(d.kind);
    int rd[3][2], wr[2][2], nr = 0, nw = 0;
    auto R = [&](int r, int c) { rd[nr][0] = r; rd[nr][1] = c; ++nr; };
    auto W = [&](int r, int c) { wr[nw][0] = r; wr[nw][1] = c; ++nw; };
    if (alg == 0) {
      switch (kind) {
        case 0: W(k, k); break;
        case 1: R(k, k); W(i, k); break;
        case 2: R(i, k); W(i, i); break;
        default: R(i, k); R(j, k); W(i, j); break;
      }
    } else {
      const int F = alg == 1 ? 4 : 8;
      if (kind == F) W(k, k);
      else if (kind == F + 1) { R(k, k); W(k, j); }
      else if (kind == F + 2) { W(k, k); W(i, k); }
      else { R(i, k); W(k, j); W(i, j); }
    }
    for (int x = 0; x < nr + nw; ++x) {
      const int r = x < nr ? rd[x][0] : wr[x - nr][0], c = x < nr ? rd[x][1] : wr[x - nr][1];
      if (!touched[id(r, c)]) {
        touched[id(r, c)] = 1;
        if (std::find(preds[t].begin(), preds[t].end(), a0 + c) == preds[t].end()) preds[t].push_back(a0 + c);
      }
    }
    for (int x = 0; x < nw; ++x) lastw[id(wr[x][0], wr[x][1])] = t;
  }
  for (int j = 0; j < p; ++j)
    for (int i = 0; i < p; ++i) {
      const int w = lastw[id(i, j)];
      auto& pr = preds[a0 + p + j];
      if (w >= 0 && std::find(pr.begin(), pr.end(), w) == pr.end()) pr.push_back(w);
    }
}

// The slab-level DAG is used for QR / LU on the register-slab kernels (TF_FINE=0 selects the
// tile-level DAG, for comparison).
bool fine_dag(int alg, int b, int ib) {
  static const int env = getenv("TF_FINE") ? atoi(getenv("TF_FINE")) : 1;
  const int on = g_slab_dag >= 0 ? g_slab_dag : env;
  if (alg == 0) return on != 0 && chol_panel_ok(b);
  return on != 0 && (alg == 1 || alg == 2) && ssrfb_reg_ok(b, ib);
}
bool fine_ok(int alg, int b, int ib) {
  return alg == 0 ? chol_panel_ok(b) : ((alg == 1 || alg == 2) && ssrfb_reg_ok(b, ib));
}

// fine: -1 = fine_dag()'s choice, 0 = tile-level, 1 = slab-level where eligible.
void build_dag(HostDag& G, int alg, int p, int b, int ib, int policy, int q = 0, int qc = -1, int e2e = 0,
               int fine = -1) {
  G.alg = alg; G.p = p; G.b = b; G.policy = policy;
  std::vector<std::vector<int>> preds;
  if (alg >= ALG_GETRS) solve_tasks(alg, p, b, ib, q, policy, G.tasks, preds);
  else if (fine < 0 ? fine_dag(alg, b, ib) : (fine > 0 && fine_ok(alg, b, ib))) {
    if (alg == 0) global_tasks_chol_panel(p, b, policy, G.tasks, preds);
    else global_tasks_fine(alg, p, b, ib, policy, G.tasks, preds, qc);
  }
  else global_tasks(alg, p, b, ib, policy, G.tasks, preds, qc);
  if (e2e) add_copy_tasks(alg, p, b, ib, G.tasks, preds);
  finalize_dag(G, preds);
}

// ------------------------------------------------------------------ multi-GPU plan
// Owner computes on a P x Q block-cyclic tile grid: tile (r,c) lives on
// rank (r mod P)*Q + (c mod Q); a task runs on the owner of the tile it writes (for
// SSRFB/SSSSM, which write (k,j) and (i,j), P = 1 keeps both on the owner of column j).
int out_row(const TaskD& d) {
  switch (d.kind) {
    case 0: case 4: case 8: return d.k;
    case 5: case 9: return d.k;
    case 2: return d.i;
    default: return d.i;
  }
}
int out_col(const TaskD& d) {
  switch (d.kind) {
    case 0: case 4: case 8: return d.k;
    case 1: case 6: case 10: return d.k;
    case 2: return d.i;
    default: return d.j;
  }
}
inline int tile_owner(int r, int c, int P, int Q) { return (r % P) * Q + (c % Q); }

struct DistPlan {
  int alg = 0, p = 0, b = 0, ib = 0, P = 1, Q = 1, nranks = 1, policy = 0;
  std::vector<TaskD> gtasks;                // global tasks, program order
  std::vector<HostDag> local;               // per rank
  std::vector<std::vector<int>> gid;        // local task -> global task (SEND/RECV: producer's)
  int max_tasks = 0, max_items = 0;
};

void build_plan(DistPlan& D, int alg, int p, int b, int ib, int P, int Q, int policy) {
  D.alg = alg; D.p = p; D.b = b; D.ib = ib; D.P = P; D.Q = Q; D.nranks = P * Q; D.policy = policy;
  const int R = D.nranks;
  std::vector<TaskD> gt;
  std::vector<std::vector<int>> gpred;
  global_tasks(alg, p, b, ib, policy, gt, gpred);
  D.gtasks = gt;
  const int nt = (int)gt.size();
  std::vector<int> own(nt);
  for (int t = 0; t < nt; ++t) own[t] = tile_owner(out_row(gt[t]), out_col(gt[t]), P, Q);
  std::vector<std::vector<int>> gsucc(nt);
  for (int t = 0; t < nt; ++t)
    for (int x : gpred[t]) gsucc[x].push_back(t);
  // consumer ranks of each producer (other than its owner)
  std::vector<std::vector<int>> peers(nt);
  for (int u = 0; u < nt; ++u) {
    std::set<int> s;
    for (int v : gsucc[u])
      if (own[v] != own[u]) s.insert(own[v]);
    peers[u].assign(s.begin(), s.end());
  }
  D.local.assign(R, HostDag());
  D.gid.assign(R, {});
  std::vector<std::vector<int>> recv_id(R, std::vector<int>());  // [rank][producer] -> local RECV id
  std::vector<std::vector<int>> send_id(R);
  for (int r = 0; r < R; ++r) {
    HostDag& L = D.local[r];
    L.alg = alg; L.p = p; L.b = b; L.policy = policy;
    std::vector<int> lid(nt, -1), sid(nt, -1), rid(nt, -1);
    auto& G = D.gid[r];
    for (int t = 0; t < nt; ++t) {
      if (own[t] == r) {
        lid[t] = (int)L.tasks.size();
        L.tasks.push_back(gt[t]);
        G.push_back(t);
        if (!peers[t].empty()) {
          sid[t] = (int)L.tasks.size();
          TaskD s{K_SEND, gt[t].k, gt[t].i, 0, (int)peers[t].size() * SEND_CHUNKS, 0, 0, gt[t].kind};
          L.tasks.push_back(s);
          G.push_back(t);
        }
      } else if (std::find(peers[t].begin(), peers[t].end(), r) != peers[t].end()) {
        rid[t] = (int)L.tasks.size();
        TaskD v{K_RECV, gt[t].k, gt[t].i, own[t], 1, 0, 0, gt[t].kind};
        L.tasks.push_back(v);
        G.push_back(t);
      }
    }
    std::vector<std::vector<int>> lpred(L.tasks.size());
    for (int v = 0; v < nt; ++v) {
      if (own[v] != r) continue;
      for (int u : gpred[v]) {
        if (own[u] == r) lpred[lid[v]].push_back(lid[u]);
        else lpred[lid[v]].push_back(rid[u]);
      }
    }
    for (int u = 0; u < nt; ++u)
      if (sid[u] >= 0) lpred[sid[u]].push_back(lid[u]);
    finalize_dag(L, lpred);
    // RECV tasks are released by the producer's rank: count that edge in the in-degree
    for (size_t t = 0; t < L.tasks.size(); ++t)
      if (L.tasks[t].kind == K_RECV) L.indeg0[t] = 1;
    recv_id[r] = rid;
    send_id[r] = sid;
  }
  // remote pushes: SEND(u) on its owner -> RECV(u) on every consumer rank
  for (int r = 0; r < R; ++r) {
    HostDag& L = D.local[r];
    for (size_t t = 0; t < L.tasks.size(); ++t) {
      TaskD& d = L.tasks[t];
      if (d.kind != K_SEND) continue;
      const int u = D.gid[r][t];
      d.j = (int)L.sends.size();
      for (int q : peers[u]) {
        const HostDag& C = D.local[q];
        const int rt = recv_id[q][u];
        const int lev = C.tasks[rt].level;
        L.sends.push_back(SendEnt{q, C.tasks[rt].item0, lev, C.qbase[lev], C.qbase[lev + 1]});
      }
    }
  }
  D.max_tasks = D.max_items = 0;
  for (auto& L : D.local) {
    D.max_tasks = std::max(D.max_tasks, (int)L.tasks.size());
    D.max_items = std::max(D.max_items, L.nitems);
  }
}

struct DevDag {
  std::shared_ptr<HostDag> h;
  TaskD* tasks = nullptr;
  int *succ_off = nullptr, *succ = nullptr, *item_task = nullptr, *indeg0 = nullptr, *roots = nullptr;
  SendEnt* sends = nullptr;
};

std::map<std::tuple<int, int, int, int, int, int, int, int, int>, DevDag> g_dags;  // (dev, alg, p, b, ib, policy, q, qc, e2e)

template <class T>
int upload(T** dst, const std::vector<T>& v) {
  TF_CUDA(cudaMalloc(dst, sizeof(T) * (v.empty() ? 1 : v.size())));
  if (!v.empty()) TF_CUDA(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return 0;
}

int upload_dag(DevDag& D) {
  int rc;
  if ((rc = upload(&D.tasks, D.h->tasks))) return rc;
  if ((rc = upload(&D.succ_off, D.h->succ_off))) return rc;
  if ((rc = upload(&D.succ, D.h->succ))) return rc;
  if ((rc = upload(&D.item_task, D.h->item_task))) return rc;
  if ((rc = upload(&D.indeg0, D.h->indeg0))) return rc;
  if ((rc = upload(&D.roots, D.h->roots))) return rc;
  if ((rc = upload(&D.sends, D.h->sends))) return rc;
  return 0;
}
void free_dag(DevDag& D) {
  cudaFree(D.tasks);
  cudaFree(D.succ_off);
  cudaFree(D.succ);
  cudaFree(D.item_task);
  cudaFree(D.indeg0);
  cudaFree(D.roots);
  cudaFree(D.sends);
  D = DevDag();
}

int get_dag(int dev, int alg, int p, int b, int ib, DevDag** out, int q = 0, int qc = -1, int e2e = 0) {
  auto key = std::make_tuple(dev, alg, p, b, ib, g_policy * 4 + (fine_dag(alg, b, ib) ? 2 : 0) + 8 * (alg == 0 ? gemm_tile_min() : 0), q, qc, e2e);
  auto it = g_dags.find(key);
  if (it != g_dags.end()) { *out = &it->second; return 0; }
  DevDag D;
  D.h = std::make_shared<HostDag>();
  build_dag(*D.h, alg, p, b, ib, g_policy, q, qc, e2e);
  int rc;
  if ((rc = upload_dag(D))) return rc;
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
void release(Buf& b) {
  if (b.p) cudaFree(b.p);
  b = Buf();
}

struct Workspace {
  Buf state, q, vx, scratch, info, trace, xt;
  Buf hostA, hostAux, hostPiv, flags;  // device buffers for tile_factor_host
  int64_t last_items = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cin = nullptr, cout = nullptr;  // tile_factor_host copy streams
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};
std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;

int g_nsm[64] = {0};
bool g_attr_set[64] = {false};
Workspace* g_last_ws = nullptr;

int device_setup(int dev) {
  if (dev >= 64) { set_err("device id %d too large", dev); return TF_ERR_UNSUPPORTED; }
  if (!g_attr_set[dev]) {
    TF_CUDA(cudaDeviceGetAttribute(&g_nsm[dev], cudaDevAttrMultiProcessorCount, dev));
    TF_LAUNCH(device_kernel_setup(smem_bytes()));
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

// State layout [indeg | items_done | head | tail | ndone abort exit]; `stride` >= the task
// count (multi-GPU: the max over ranks, so `tail` sits at the same offset on every rank).
void fill_sched(Sched& S, const HostDag& H, const DevDag& D, int* st, int* q, int stride = -1) {
  const int nt = (int)H.tasks.size();
  const int ns = ((stride < 0 ? nt : stride) + 3) & ~3;  // head/tail 16-byte aligned (vector loads)
  S.tasks = D.tasks;
  S.succ_off = D.succ_off;
  S.succ = D.succ;
  S.item_task = D.item_task;
  S.ntasks = nt;
  S.nitems = H.nitems;
  for (int l = 0; l <= NLEV; ++l) S.qbase[l] = H.qbase[l];
  S.indeg = st;
  S.items_done = st + ns;
  S.head = st + 2 * ns;
  S.tail = S.head + NLEV;
  S.ndone = S.tail + NLEV;
  S.abort_flag = S.ndone + 1;
  S.exit_count = S.ndone + 2;
  S.q = q;
  S.trace = nullptr;
  S.trace_cap = 0;
}

// Single-GPU scheduler watchdog: no CTA of the one-GPU kernel waits for a specific task,
// so the only way it can stall is a lost queue push (a bug); if no item can be popped for
// TF_WATCHDOG_S seconds (default 60, far above the longest item, ~3.3 ms) the kernel
// aborts with info = -1 instead of hanging the GPU.  0 disables it.
long long watchdog_ns() {
  const char* e = getenv("TF_WATCHDOG_S");
  const double s = e ? atof(e) : 60.0;
  return s > 0 ? (long long)(s * 1e9) : 0;
}

// m_rows >= 0: QR / LU of an m_rows x n matrix (p = m_rows/b tile rows, n/b tile columns).
// copy_flags (tile_factor_host): [p] arrive flags, [p] done flags, [1] arrive cursor; the
// DAG then has ARRIVE / DONE tasks (add_copy_tasks).
int run_factorization(int alg, int64_t n, int64_t b, int64_t ib, double* dA, double* aux, int32_t* ipiv,
                      int32_t* d_info, cudaStream_t stream, double* X = nullptr, int q = 0, int nopiv = 0,
                      int64_t m_rows = -1, int* copy_flags = nullptr) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  int rc;
  if ((rc = device_setup(dev))) return rc;
  const int p = (int)((m_rows >= 0 ? m_rows : n) / b);
  const int qc = m_rows >= 0 ? (int)(n / b) : -1;
  DevDag* D;
  if ((rc = get_dag(dev, alg, p, (int)b, (int)ib, &D, q, qc, copy_flags ? 1 : 0))) return rc;
  const HostDag& H = *D->h;
  Workspace& W = g_ws[std::make_pair(dev, stream)];
  W.stream = stream;
  const int nt = (int)H.tasks.size();
  const int ctas = g_ctas > 0 ? g_ctas : g_nsm[dev];
  const size_t state_ints = (size_t)2 * (nt + 4) + 2 * NLEV + 8;
  if ((rc = ensure(W.state, state_ints * sizeof(int)))) return rc;
  if ((rc = ensure(W.q, (size_t)H.nitems * sizeof(int)))) return rc;
  if (alg != 0 && alg != ALG_LUN && (rc = ensure(W.vx, (size_t)p * b * b * sizeof(double)))) return rc;
  const size_t scr = scr_stride_for((int)b, (int)ib);
  if ((rc = ensure(W.scratch, scr * ctas * sizeof(double)))) return rc;
  if ((rc = ensure(W.info, 64))) return rc;
  if (g_trace_cap > 0 && (rc = ensure(W.trace, (size_t)H.nitems * 5 * sizeof(long long)))) return rc;
  static Runs R;  // large; guarded by g_mu
  memset(&R, 0, sizeof(R));
  R.nruns = 1;
  Sched& S = R.r[0].S;
  fill_sched(S, H, *D, (int*)W.state.p, (int*)W.q.p);
  S.trace = g_trace_cap > 0 ? (long long*)W.trace.p : nullptr;
  S.trace_cap = g_trace_cap > 0 ? H.nitems : 0;
  W.last_items = g_trace_cap > 0 ? H.nitems : 0;
  Prob& P = R.r[0].P;
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
  P.X = X;
  P.q = q;
  P.nopiv = nopiv;
  if (copy_flags) {
    S.arrive_flags = copy_flags;
    S.done_flags = copy_flags + p;
    S.arrive_next = copy_flags + 2 * p;
    S.arrive_task0 = (int)H.tasks.size() - 2 * p;
    S.narrive = p;
  }
  R.r[0].D.timeout_ns = watchdog_ns();
  TF_LAUNCH(launch_sched_reset(S, D->indeg0, H.nitems, P.info, stream));
  TF_LAUNCH(launch_sched_seed(S, D->roots, (int)H.roots.size(), stream));
  TF_LAUNCH(launch_persistent(R, ctas, smem_bytes(), stream, false));
  g_last_ws = &W;
  return 0;
}

// ------------------------------------------------------------------ multi-GPU ranks
// One DistRank per (rank, process): the rank's local DAG on the device, its symmetric
// block (sync flags, scheduler state, queue, receive cache) and the peers' mapped blocks.
struct DistRank {
  std::shared_ptr<DistPlan> plan;
  int rank = 0, dev = 0;
  int64_t n = 0;
  DevDag dag;
  Buf sym, vx, scratch, ptab;
  size_t off_state = 0, off_q = 0, off_ctile = 0, off_cstrip = 0, off_cpiv = 0, sym_bytes = 0;
  char* peer_sym[TF_MAX_RANKS] = {nullptr};
  bool ipc_opened[TF_MAX_RANKS] = {false};
  const void* key[3] = {nullptr, nullptr, nullptr};
  int epoch = 0;
  bool connected = false;
};

std::map<std::tuple<int, int, int, int, int, int, int, int>, std::shared_ptr<DistPlan>> g_plans;

std::shared_ptr<DistPlan> get_plan(int alg, int p, int b, int ib, int P, int Q) {
  auto key = std::make_tuple(alg, p, b, ib, P, Q, g_policy, 0);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return it->second;
  auto pl = std::make_shared<DistPlan>();
  build_plan(*pl, alg, p, b, ib, P, Q, g_policy);
  g_plans[key] = pl;
  return pl;
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// local storage: rank's tiles (i,j) at (i/P + (j/Q)*pl) with pl = ceil(p/P) rows
inline int64_t loc_rows(int p, int P) { return (p + P - 1) / P; }
inline int64_t loc_cols(int p, int Q) { return (p + Q - 1) / Q; }

int check_dist_args(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q) {
  if (alg < 0 || alg > 2) { set_err("alg must be 0 (chol), 1 (qr) or 2 (lu)"); return -1; }
  if (n <= 0) { set_err("n must be > 0"); return -2; }
  if (b <= 0 || n % b || b > TF_MAX_B) { set_err("b must be > 0 and divide n"); return -3; }
  if (b % 4) { set_err("multi-GPU needs b %% 4 == 0 (16-byte payload chunks)"); return -3; }
  if (ib <= 0 || b % ib) { set_err("ib must be > 0 and divide b"); return -4; }
  if (P <= 0 || Q <= 0 || P * Q > TF_MAX_RANKS) { set_err("P*Q must be in [1, %d]", TF_MAX_RANKS); return -5; }
  if (alg != 0 && P != 1) { set_err("QR/LU use a 1 x Q column-cyclic grid (P must be 1)"); return -5; }
  return 0;
}

int dist_create(DistRank& X, int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, int rank) {
  X.plan = get_plan(alg, (int)(n / b), (int)b, (int)ib, P, Q);
  X.rank = rank;
  X.n = n;
  TF_CUDA(cudaGetDevice(&X.dev));
  int rc;
  if ((rc = device_setup(X.dev))) return rc;
  const DistPlan& pl = *X.plan;
  const int p = pl.p;
  const size_t bb = (size_t)b * b;
  const size_t nslots = pl.nranks > 1 ? (size_t)p * (p + 1) / 2 : 0;
  X.off_state = SY_INTS * sizeof(int);
  const size_t state_ints = (size_t)2 * (pl.max_tasks + 4) + 2 * NLEV + 8;
  X.off_q = align256(X.off_state + state_ints * sizeof(int));
  X.off_ctile = align256(X.off_q + (size_t)pl.max_items * sizeof(int));
  X.off_cstrip = X.off_ctile + nslots * bb * sizeof(double);
  X.off_cpiv = X.off_cstrip + (alg != 0 ? nslots * ib * b * sizeof(double) : 0);
  X.sym_bytes = align256(X.off_cpiv + (alg == 2 ? nslots * b * sizeof(int) : 0));
  if ((rc = ensure(X.sym, X.sym_bytes))) return rc;
  TF_CUDA(cudaMemset(X.sym.p, 0, X.off_ctile));
  TF_CUDA(cudaDeviceSynchronize());  // zeroed before the handle reaches any peer
  if (alg != 0 && (rc = ensure(X.vx, (size_t)loc_cols(p, Q) * bb * sizeof(double)))) return rc;
  X.dag.h = std::shared_ptr<HostDag>(X.plan, &X.plan->local[rank]);
  if ((rc = upload_dag(X.dag))) return rc;
  for (int r = 0; r < TF_MAX_RANKS; ++r) X.peer_sym[r] = nullptr;
  X.peer_sym[rank] = (char*)X.sym.p;
  return 0;
}

void dist_destroy(DistRank& X) {
  for (int r = 0; r < TF_MAX_RANKS; ++r)
    if (X.ipc_opened[r] && X.peer_sym[r]) cudaIpcCloseMemHandle(X.peer_sym[r]);
  release(X.sym);
  release(X.vx);
  release(X.scratch);
  release(X.ptab);
  free_dag(X.dag);
}

// Pointer tables for this call's local buffers (rebuilt only when the buffers change).
int dist_tables(DistRank& X, double* dA, double* dAux, int32_t* dPiv, cudaStream_t stream) {
  if (X.key[0] == dA && X.key[1] == dAux && X.key[2] == dPiv && X.ptab.p) return 0;
  const DistPlan& pl = *X.plan;
  const int p = pl.p, P = pl.P, Q = pl.Q;
  const size_t bb = (size_t)pl.b * pl.b, sb = (size_t)pl.ib * pl.b;
  const int64_t lr = loc_rows(p, P);
  const size_t np2 = (size_t)p * p;
  std::vector<uintptr_t> tab(3 * np2 + p, 0);
  char* sym = (char*)X.sym.p;
  for (int j = 0; j < p; ++j)
    for (int i = 0; i < p; ++i) {
      const size_t e = i + (size_t)j * p;
      const size_t loc = (size_t)(i / P) + (size_t)(j / Q) * lr;
      if (tile_owner(i, j, P, Q) == X.rank) {
        tab[e] = (uintptr_t)(dA + loc * bb);
        if (dAux) tab[np2 + e] = (uintptr_t)(dAux + loc * sb);
        if (dPiv) tab[2 * np2 + e] = (uintptr_t)(dPiv + loc * pl.b);
      } else if (i >= j && pl.nranks > 1) {
        const long long s = cache_slot(i, j, p);
        tab[e] = (uintptr_t)(sym + X.off_ctile + s * bb * sizeof(double));
        if (pl.alg != 0) tab[np2 + e] = (uintptr_t)(sym + X.off_cstrip + s * sb * sizeof(double));
        if (pl.alg == 2) tab[2 * np2 + e] = (uintptr_t)(sym + X.off_cpiv + s * pl.b * sizeof(int));
      }
    }
  for (int k = 0; k < p; ++k) {
    if (pl.alg == 0) continue;
    if (tile_owner(k, k, P, Q) == X.rank) tab[3 * np2 + k] = (uintptr_t)((double*)X.vx.p + (size_t)(k / Q) * bb);
    else tab[3 * np2 + k] = tab[k + (size_t)k * p];  // the cache slot of (k,k) holds the V_kk / L_kk copy
  }
  int rc;
  if ((rc = ensure(X.ptab, tab.size() * sizeof(uintptr_t)))) return rc;
  TF_CUDA(cudaMemcpyAsync(X.ptab.p, tab.data(), tab.size() * sizeof(uintptr_t), cudaMemcpyHostToDevice, stream));
  TF_CUDA(cudaStreamSynchronize(stream));  // `tab` is pageable and goes out of scope
  X.key[0] = dA;
  X.key[1] = dAux;
  X.key[2] = dPiv;
  return 0;
}

long long dist_timeout_ns() {
  const char* e = getenv("TF_DIST_TIMEOUT_S");
  const double s = e ? atof(e) : 120.0;
  return s > 0 ? (long long)(s * 1e9) : 0;
}

// Fill one rank's RankRun and enqueue its reset + seed kernels.
int dist_prepare(DistRank& X, RankRun& RR, int cta0, int nctas, double* dA, double* dAux, int32_t* dPiv,
                 int32_t* d_info, cudaStream_t stream) {
  const DistPlan& pl = *X.plan;
  int rc;
  if ((rc = dist_tables(X, dA, dAux, dPiv, stream))) return rc;
  const size_t scr = scr_stride_for(pl.b, pl.ib);
  if ((rc = ensure(X.scratch, scr * nctas * sizeof(double)))) return rc;
  const HostDag& H = *X.dag.h;
  char* sym = (char*)X.sym.p;
  int* sync = (int*)sym;
  Sched& S = RR.S;
  fill_sched(S, H, X.dag, (int*)(sym + X.off_state), (int*)(sym + X.off_q), pl.max_tasks);
  S.abort_flag = sync + SY_ABORT;
  Prob& P = RR.P;
  P.A = dA;
  P.aux = dAux;
  P.ipiv = dPiv;
  P.vx = (double*)X.vx.p;
  P.scratch = (double*)X.scratch.p;
  P.scr_stride = scr;
  P.n = (int)X.n;
  P.b = pl.b;
  P.ib = pl.ib;
  P.p = pl.p;
  P.info = sync + SY_LINFO;
  Dist& D = RR.D;
  const size_t np2 = (size_t)pl.p * pl.p;
  double* const* tab = (double* const*)X.ptab.p;
  D.nranks = pl.nranks;
  D.rank = X.rank;
  D.epoch = ++X.epoch;
  D.cta0 = cta0;
  D.nctas = nctas;
  D.tptr = tab;
  D.sptr = tab + np2;
  D.pptr = (int* const*)(tab + 2 * np2);
  D.vptr = tab + 3 * np2;
  D.sends = X.dag.sends;
  for (int r = 0; r < TF_MAX_RANKS; ++r) D.peer_sym[r] = X.peer_sym[r];
  D.off_tail = X.off_state + ((size_t)2 * ((pl.max_tasks + 3) & ~3) + NLEV) * sizeof(int);
  D.off_q = X.off_q;
  D.off_ctile = X.off_ctile;
  D.off_cstrip = X.off_cstrip;
  D.off_cpiv = X.off_cpiv;
  D.sym_bytes = X.sym_bytes;
  D.user_info = d_info;
  D.timeout_ns = dist_timeout_ns();
  TF_LAUNCH(launch_sched_reset(S, X.dag.indeg0, H.nitems, P.info, stream));
  TF_LAUNCH(launch_sched_seed(S, X.dag.roots, (int)H.roots.size(), stream));
  return 0;
}

struct EmuKey {
  int dev, alg;
  int64_t n, b, ib;
  int P, Q, policy;
  bool operator<(const EmuKey& o) const {
    return std::tie(dev, alg, n, b, ib, P, Q, policy) < std::tie(o.dev, o.alg, o.n, o.b, o.ib, o.P, o.Q, o.policy);
  }
};
std::map<EmuKey, std::vector<std::unique_ptr<DistRank>>> g_emu;
std::set<DistRank*> g_handles;

}  // namespace

// ====================================================================================
// C-ABI
// ====================================================================================
struct tf_dist_s {
  DistRank r;
};

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

// Solve / apply entry points (NEXT-3): X (n x nrhs, ld ldx, device) is packed into library
// BDL scratch, the solve DAG runs on the persistent scheduler, X is unpacked; all async on
// `stream` (the scratch is per (device, stream), so calls on one stream serialize).
static int run_solve(int alg, int64_t n, int64_t b, int64_t ib, const double* dF, const double* dAux,
                     const int32_t* dIpiv, int64_t nrhs, double* dX, int64_t ldx, tf_stream_t stream) {
  int rc = check_args(n, b, ib, dF);
  if (rc) return rc;
  if (!dAux) { set_err("null T / L-strip pointer"); return -5; }
  const bool lu = alg == ALG_GETRS || alg == ALG_LUN;
  if (lu && !dIpiv) { set_err("null ipiv pointer"); return -6; }
  if (nrhs < 0) { set_err("nrhs < 0"); return -7; }
  if (nrhs == 0) return 0;
  if (!dX) { set_err("null X pointer"); return -8; }
  if (ldx < n) { set_err("ldx < n"); return -9; }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t q = (nrhs + b - 1) / b;
  if (q > (1 << 16)) { set_err("too many right-hand sides"); return -7; }
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  Workspace* W;
  {
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    W = &g_ws[std::make_pair(dev, s)];
    if ((rc = ensure(W->xt, (size_t)n * q * b * sizeof(double)))) return rc;
  }
  double* Xt = (double*)W->xt.p;
  TF_LAUNCH(launch_xpack(n, nrhs, ldx, b, q, dX, Xt, 0, s));
  if ((rc = run_factorization(alg, n, b, ib, const_cast<double*>(dF), const_cast<double*>(dAux),
                              const_cast<int32_t*>(dIpiv), nullptr, s, Xt, (int)q)))
    return rc;
  TF_LAUNCH(launch_xpack(n, nrhs, ldx, b, q, dX, Xt, 1, s));
  return 0;
}

int tile_getrs(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dLs, const int32_t* dIpiv,
               int64_t nrhs, double* dX, int64_t ldx, tf_stream_t stream) {
  return run_solve(ALG_GETRS, n, b, ib, dF, dLs, dIpiv, nrhs, dX, ldx, stream);
}
int tile_ormqr(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dT, int64_t nrhs, double* dX,
               int64_t ldx, tf_stream_t stream) {
  return run_solve(ALG_ORMQR, n, b, ib, dF, dT, nullptr, nrhs, dX, ldx, stream);
}
int tile_qrs(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dT, int64_t nrhs, double* dX,
             int64_t ldx, tf_stream_t stream) {
  return run_solve(ALG_QRS, n, b, ib, dF, dT, nullptr, nrhs, dX, ldx, stream);
}
int tile_lu_apply_N(int64_t n, int64_t b, int64_t ib, const double* dF, const double* dLs, const int32_t* dIpiv,
                    int64_t nrhs, double* dX, int64_t ldx, tf_stream_t stream) {
  return run_solve(ALG_LUN, n, b, ib, dF, dLs, dIpiv, nrhs, dX, ldx, stream);
}
int tile_lu_nopiv(int64_t n, int64_t b, int64_t ib, double* dA, double* dLs, int32_t* dIpiv, int32_t* d_info,
                  tf_stream_t stream) {
  int rc = check_args(n, b, ib, dA);
  if (rc) return rc;
  if (!dLs) { set_err("null L-strip pointer"); return -5; }
  if (!dIpiv) { set_err("null ipiv pointer"); return -6; }
  return run_factorization(2, n, b, ib, dA, dLs, dIpiv, d_info, (cudaStream_t)stream, nullptr, 0, 1);
}

// Rectangular QR / LU (NEXT-4).
static int check_mn(int64_t m, int64_t n, int64_t b, int64_t ib, const void* dA) {
  if (m <= 0) { set_err("m must be > 0"); return -1; }
  if (n <= 0) { set_err("n must be > 0"); return -2; }
  if (b <= 0 || m % b || n % b || b > TF_MAX_B) { set_err("b must be > 0 and divide m and n"); return -3; }
  if (ib <= 0 || b % ib) { set_err("ib must be > 0 and divide b"); return -4; }
  if (!dA) { set_err("null matrix pointer"); return -5; }
  if ((m / b) * (n / b) > (int64_t)1 << 24) { set_err("too many tiles"); return -1; }
  return 0;
}
int tile_qr_mn(int64_t m, int64_t n, int64_t b, int64_t ib, double* dA, double* dT, tf_stream_t stream) {
  int rc = check_mn(m, n, b, ib, dA);
  if (rc) return rc;
  if (!dT) { set_err("null T pointer"); return -6; }
  return run_factorization(1, n, b, ib, dA, dT, nullptr, nullptr, (cudaStream_t)stream, nullptr, 0, 0, m);
}
int tile_lu_mn(int64_t m, int64_t n, int64_t b, int64_t ib, double* dA, double* dLs, int32_t* dIpiv,
               int32_t* d_info, tf_stream_t stream) {
  int rc = check_mn(m, n, b, ib, dA);
  if (rc) return rc;
  if (!dLs) { set_err("null L-strip pointer"); return -6; }
  if (!dIpiv) { set_err("null ipiv pointer"); return -7; }
  return run_factorization(2, n, b, ib, dA, dLs, dIpiv, d_info, (cudaStream_t)stream, nullptr, 0, 0, m);
}
size_t tile_mn_aux_elems(int64_t m, int64_t n, int64_t b, int64_t ib) {
  if (m <= 0 || n <= 0 || b <= 0 || m % b || n % b) return 0;
  const size_t p = m / b, q = n / b;
  return p * (p < q ? p : q) * (size_t)ib * b;
}
size_t tile_mn_ipiv_elems(int64_t m, int64_t n, int64_t b) {
  if (m <= 0 || n <= 0 || b <= 0 || m % b || n % b) return 0;
  const size_t p = m / b, q = n / b;
  return p * (p < q ? p : q) * (size_t)b;
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
  TF_LAUNCH(launch_pack(m, n, b, const_cast<double*>(dDense), dTiles, 0, stream));
  return 0;
}

int tile_unpack(int64_t m, int64_t n, int64_t b, const double* dTiles, double* dDense, tf_stream_t stream) {
  if (m <= 0 || n <= 0) return -1;
  if (b <= 0 || m % b || n % b) return -3;
  if (!dTiles) return -4;
  if (!dDense) return -5;
  TF_LAUNCH(launch_pack(m, n, b, dDense, const_cast<double*>(dTiles), 1, stream));
  return 0;
}

// Stream memory operations (driver API, through the runtime's entry-point query so the
// library keeps no link dependency on libcuda): the H2D copy stream writes a column's
// arrival flag after its bytes; the D2H copy stream waits on a column's done flag.
typedef int (*pfn_stream_value32)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
static pfn_stream_value32 g_write32 = nullptr, g_wait32 = nullptr;
static int stream_memops() {
  if (g_write32 && g_wait32) return 0;
  cudaDriverEntryPointQueryResult q1, q2;
  void *w = nullptr, *t = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &q2) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !t) {
    cudaGetLastError();
    set_err("stream memory operations unavailable");
    return TF_ERR_UNSUPPORTED;
  }
  g_write32 = (pfn_stream_value32)w;
  g_wait32 = (pfn_stream_value32)t;
  return 0;
}

// End-to-end host-buffer path with the copies overlapped with the factorization: tile
// column j goes host -> device on one copy stream (then its arrival flag), the DAG's first
// task touching column j waits for that flag (ARRIVE(j)), and as soon as every tile of
// column j is final (DONE(j)) a second copy stream brings it back while the trailing
// updates run.  TF_E2E_SERIAL=1 selects the serial copy / factor / copy path.
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
    std::lock_guard<std::recursive_mutex> lk(g_mu);
    W = &g_ws[std::make_pair(dev, s)];
  }
  const size_t an = (size_t)n * n;
  const size_t xn = kind == 0 ? 0 : tile_qr_t_elems(n, b, ib);
  const size_t pn = kind == 2 ? tile_lu_ipiv_elems(n, b) : 0;
  const int64_t p = n / b;
  if ((rc = ensure(W->hostA, an * sizeof(double) + 64))) return rc;
  if (xn && (rc = ensure(W->hostAux, xn * sizeof(double)))) return rc;
  if (pn && (rc = ensure(W->hostPiv, pn * sizeof(int32_t) + 64))) return rc;
  double* dA = (double*)W->hostA.p;
  double* dAux = (double*)W->hostAux.p;
  int32_t* dPiv = (int32_t*)W->hostPiv.p;
  int32_t* dInfo = (int32_t*)((char*)W->hostA.p + an * sizeof(double));
  const char* ser = getenv("TF_E2E_SERIAL");
  if ((ser && atoi(ser)) || stream_memops() != 0) {
    TF_CUDA(cudaMemcpyAsync(dA, hA, an * sizeof(double), cudaMemcpyHostToDevice, s));
    if (kind == 0) rc = tile_chol(n, b, ib, dA, dInfo, stream);
    else if (kind == 1) rc = tile_qr(n, b, ib, dA, dAux, stream);
    else rc = tile_lu(n, b, ib, dA, dAux, dPiv, dInfo, stream);
    if (rc) return rc;
    TF_CUDA(cudaMemcpyAsync(hA, dA, an * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (hAux && xn) TF_CUDA(cudaMemcpyAsync(hAux, dAux, xn * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (hIpiv && pn) TF_CUDA(cudaMemcpyAsync(hIpiv, dPiv, pn * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (hInfo) {
      if (kind == 1) *hInfo = 0;
      else TF_CUDA(cudaMemcpyAsync(hInfo, dInfo, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    TF_CUDA(cudaStreamSynchronize(s));
    return 0;
  }
  if (!W->cin) {
    TF_CUDA(cudaStreamCreateWithFlags(&W->cin, cudaStreamNonBlocking));
    TF_CUDA(cudaStreamCreateWithFlags(&W->cout, cudaStreamNonBlocking));
    TF_CUDA(cudaEventCreateWithFlags(&W->ev0, cudaEventDisableTiming));
    TF_CUDA(cudaEventCreateWithFlags(&W->ev1, cudaEventDisableTiming));
  }
  if ((rc = ensure(W->flags, (size_t)(2 * p + 4) * sizeof(int)))) return rc;
  int* flags = (int*)W->flags.p;
  // flags reset on the compute stream, before either copy stream touches them
  TF_CUDA(cudaMemsetAsync(flags, 0, (size_t)(2 * p + 4) * sizeof(int), s));
  TF_CUDA(cudaEventRecord(W->ev0, s));
  TF_CUDA(cudaStreamWaitEvent(W->cin, W->ev0, 0));
  TF_CUDA(cudaStreamWaitEvent(W->cout, W->ev0, 0));
  const size_t bb = (size_t)b * b, colA = (size_t)p * bb;
  // Cholesky reads and writes only the lower tiles (i >= j) of column j
  auto col_off = [&](int64_t j) { return kind == 0 ? (size_t)j * colA + (size_t)j * bb : (size_t)j * colA; };
  auto col_len = [&](int64_t j) { return kind == 0 ? (size_t)(p - j) * bb : colA; };
  for (int64_t j = 0; j < p; ++j) {
    TF_CUDA(cudaMemcpyAsync(dA + col_off(j), hA + col_off(j), col_len(j) * sizeof(double), cudaMemcpyHostToDevice,
                            W->cin));
    if (g_write32(W->cin, (unsigned long long)(uintptr_t)(flags + j), 1u, 0u) != 0) {
      set_err("cuStreamWriteValue32 failed");
      return TF_ERR_CUDA;
    }
  }
  if ((rc = run_factorization(kind, n, b, ib, dA, kind ? dAux : nullptr, kind == 2 ? dPiv : nullptr,
                              kind == 1 ? nullptr : dInfo, s, nullptr, 0, 0, -1, flags)))
    return rc;
  for (int64_t j = 0; j < p; ++j) {
    if (g_wait32(W->cout, (unsigned long long)(uintptr_t)(flags + p + j), 1u, 0u /* GEQ */) != 0) {
      set_err("cuStreamWaitValue32 failed");
      return TF_ERR_CUDA;
    }
    TF_CUDA(cudaMemcpyAsync(hA + col_off(j), dA + col_off(j), col_len(j) * sizeof(double), cudaMemcpyDeviceToHost,
                            W->cout));
    // T strips (i, j), i >= j; L strips (i, j), i > j; pivot vectors (i, j), i >= j (the
    // ones the factorization writes)
    const int64_t x0 = kind == 2 ? j + 1 : j;
    const size_t sx = (size_t)(x0 + j * p) * ib * b, nx = (size_t)(p - x0) * ib * b;
    const size_t sp = (size_t)(j + j * p) * b, npv = (size_t)(p - j) * b;
    if (hAux && xn && nx)
      TF_CUDA(cudaMemcpyAsync(hAux + sx, dAux + sx, nx * sizeof(double), cudaMemcpyDeviceToHost, W->cout));
    if (hIpiv && pn)
      TF_CUDA(cudaMemcpyAsync(hIpiv + sp, dPiv + sp, npv * sizeof(int32_t), cudaMemcpyDeviceToHost, W->cout));
  }
  TF_CUDA(cudaEventRecord(W->ev1, s));  // the factorization (and its info) finished
  TF_CUDA(cudaStreamWaitEvent(W->cout, W->ev1, 0));
  if (hInfo) {
    if (kind == 1) *hInfo = 0;
    else TF_CUDA(cudaMemcpyAsync(hInfo, dInfo, sizeof(int32_t), cudaMemcpyDeviceToHost, W->cout));
  }
  // the caller's stream orders after both copy streams (its events time the whole path)
  TF_CUDA(cudaEventRecord(W->ev0, W->cin));
  TF_CUDA(cudaStreamWaitEvent(s, W->ev0, 0));
  TF_CUDA(cudaEventRecord(W->ev1, W->cout));
  TF_CUDA(cudaStreamWaitEvent(s, W->ev1, 0));
  TF_CUDA(cudaStreamSynchronize(s));
  return 0;
}

void tile_set_policy(int policy) { g_policy = (policy == 0) ? 0 : 1; }
void tile_set_slab_dag(int on) { g_slab_dag = on < 0 ? -1 : (on ? 1 : 0); }
void tile_set_gemm_tile_min(int min_tiles) { g_gemm_tile_min = min_tiles < 0 ? -1 : min_tiles; }
void tile_set_trace(int64_t cap) { g_trace_cap = cap > 0 ? cap : 0; }
void tile_set_ctas(int ctas) { g_ctas = ctas > 0 ? ctas : 0; }

int64_t tile_trace_fetch(int64_t* rec, int64_t cap) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
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
  if (alg < 0 || alg > ALG_LUN || p <= 0) return -1;
  HostDag G;
  build_dag(G, alg, (int)p, 128, 32, policy, alg >= ALG_GETRS ? 1 : 0, -1, 0, /*fine=*/0);
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

int64_t tile_dag_export_slab(int alg, int64_t p, int64_t b, int64_t ib, int policy, int32_t* kind, int32_t* k,
                             int32_t* i, int32_t* j, int32_t* slab, int32_t* level, int64_t cap, int64_t* succ_off,
                             int32_t* succ, int64_t succ_cap, int64_t* nedges) {
  if (alg < 0 || alg > 2 || p <= 0 || !fine_ok(alg, (int)b, (int)ib)) return -1;
  HostDag G;
  build_dag(G, alg, (int)p, (int)b, (int)ib, policy, 0, -1, 0, /*fine=*/1);
  const int64_t nt = (int64_t)G.tasks.size();
  for (int64_t t = 0; t < nt && t < cap; ++t) {
    if (kind) kind[t] = G.tasks[t].kind;
    if (k) k[t] = G.tasks[t].k;
    if (i) i[t] = G.tasks[t].i;
    if (j) j[t] = G.tasks[t].j;
    if (slab) slab[t] = G.tasks[t].pad;
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
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  int rc;
  if ((rc = device_setup(dev))) return rc;
  Workspace& W = g_ws[std::make_pair(dev, s)];
  const int items = items_of(kind, (int)b, (int)ib);
  const size_t scr = scr_stride_for((int)b, (int)ib);
  if ((rc = ensure(W.scratch, scr * items * sizeof(double)))) return rc;
  if ((rc = ensure(W.vx, (size_t)b * b * sizeof(double)))) return rc;
  double* vx = (double*)W.vx.p;
  if (kind == 5 || kind == 9) TF_LAUNCH(launch_unit_lower(t0, vx, (int)b, s));
  TF_LAUNCH(launch_tk(kind, (int)b, (int)ib, t0, t1, t2, aux, ipiv, vx, (double*)W.scratch.p, scr, d_info, items,
                      smem_bytes(), s));
  return 0;
}

// ---------------------------------------------------------------- multi-GPU
int64_t tile_dist_local_elems(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, int which) {
  if (check_dist_args(alg, n, b, ib, P, Q)) return -1;
  const int p = (int)(n / b);
  const int64_t tiles = loc_rows(p, P) * loc_cols(p, Q);
  switch (which) {
    case 0: return tiles * b * b;
    case 1: return alg == 0 ? 0 : tiles * ib * b;
    case 2: return alg == 2 ? tiles * b : 0;
    default: return -1;
  }
}

int tile_dist_owner(int64_t i, int64_t j, int P, int Q) {
  if (i < 0 || j < 0 || P <= 0 || Q <= 0) return -1;
  return tile_owner((int)i, (int)j, P, Q);
}

int64_t tile_dist_plan_export(int alg, int64_t p, int P, int Q, int rank, int32_t* kind, int32_t* k, int32_t* i,
                              int32_t* j, int32_t* link, int32_t* gid, int64_t cap, int64_t* succ_off, int32_t* succ,
                              int64_t succ_cap, int32_t* send_peer, int32_t* send_task, int64_t send_cap,
                              int64_t* nedges, int64_t* nsends) {
  if (check_dist_args(alg, p * 4, 4, 4, P, Q) || rank < 0 || rank >= P * Q) return -1;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  auto pl = get_plan(alg, (int)p, 4, 4, P, Q);
  const HostDag& L = pl->local[rank];
  const int64_t nt = (int64_t)L.tasks.size();
  for (int64_t t = 0; t < nt && t < cap; ++t) {
    const TaskD& d = L.tasks[t];
    if (kind) kind[t] = d.kind;
    if (k) k[t] = d.k;
    if (i) i[t] = d.i;
    if (j) j[t] = pl->gtasks[pl->gid[rank][t]].j;
    if (link) link[t] = d.kind == K_SEND ? d.j : (d.kind == K_RECV ? d.j : -1);
    if (gid) gid[t] = pl->gid[rank][t];
  }
  if (succ_off && cap >= nt)
    for (int64_t t = 0; t <= nt; ++t) succ_off[t] = L.succ_off[t];
  const int64_t ne = (int64_t)L.succ.size();
  if (succ)
    for (int64_t e = 0; e < ne && e < succ_cap; ++e) succ[e] = L.succ[e];
  if (nedges) *nedges = ne;
  const int64_t ns = (int64_t)L.sends.size();
  for (int64_t e = 0; e < ns && e < send_cap; ++e) {
    const SendEnt& s = L.sends[e];
    if (send_peer) send_peer[e] = s.peer;
    if (send_task) send_task[e] = pl->local[s.peer].item_task[s.item];
  }
  if (nsends) *nsends = ns;
  return nt;
}

int tile_dist_open(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, int rank, void* ipc_out,
                   tf_dist_t* out) {
  int rc = check_dist_args(alg, n, b, ib, P, Q);
  if (rc) return rc;
  if (rank < 0 || rank >= P * Q) { set_err("rank out of range"); return -7; }
  if (!out) return -9;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  auto* h = new tf_dist_s();
  if ((rc = dist_create(h->r, alg, n, b, ib, P, Q, rank))) {
    dist_destroy(h->r);
    delete h;
    return rc;
  }
  if (ipc_out) {
    cudaIpcMemHandle_t hd;
    if (cudaIpcGetMemHandle(&hd, h->r.sym.p) != cudaSuccess) {
      set_err("cudaIpcGetMemHandle failed");
      dist_destroy(h->r);
      delete h;
      return TF_ERR_CUDA;
    }
    memcpy(ipc_out, &hd, sizeof(hd));
  }
  g_handles.insert(&h->r);
  *out = h;
  return 0;
}

int tile_dist_ipc_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int tile_dist_connect(tf_dist_t h, const void* all_ipc) {
  if (!h) return -1;
  if (!all_ipc) return -2;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  DistRank& X = h->r;
  const int R = X.plan->nranks;
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  for (int r = 0; r < R; ++r) {
    if (r == X.rank) continue;
    int can = 0;
    cudaIpcMemHandle_t hd;
    memcpy(&hd, (const char*)all_ipc + r * hb, hb);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      set_err("cudaIpcOpenMemHandle(rank %d): %s (peer access %d)", r, cudaGetErrorString(e), can);
      return TF_ERR_CUDA;
    }
    X.peer_sym[r] = (char*)p;
    X.ipc_opened[r] = true;
  }
  X.connected = true;
  return 0;
}

int tile_dist_factor(tf_dist_t h, double* dA_loc, double* dAux_loc, int32_t* dIpiv_loc, int32_t* d_info,
                     tf_stream_t stream) {
  if (!h) return -1;
  DistRank& X = h->r;
  if (!dA_loc) { set_err("null local matrix"); return -2; }
  if (X.plan->alg != 0 && !dAux_loc) { set_err("null local T/L strips"); return -3; }
  if (X.plan->alg == 2 && !dIpiv_loc) { set_err("null local ipiv"); return -4; }
  if (!d_info) { set_err("null d_info"); return -5; }
  if (X.plan->nranks > 1 && !X.connected) { set_err("tile_dist_connect not called"); return TF_ERR_UNSUPPORTED; }
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  cudaStream_t s = (cudaStream_t)stream;
  // the start/end barriers need every CTA co-resident: at most one CTA per SM
  const int ctas = g_ctas > 0 ? std::min(g_ctas, g_nsm[X.dev]) : g_nsm[X.dev];
  static Runs R;
  memset(&R, 0, sizeof(R));
  R.nruns = 1;
  int rc;
  if ((rc = dist_prepare(X, R.r[0], 0, ctas, dA_loc, dAux_loc, dIpiv_loc, d_info, s))) return rc;
  TF_LAUNCH(launch_persistent(R, ctas, smem_bytes(), s, true));
  return 0;
}

int tile_dist_probe(tf_dist_t h, int peer, int32_t value, tf_stream_t stream) {
  if (!h) return -1;
  DistRank& X = h->r;
  if (peer < 0 || peer >= X.plan->nranks || !X.peer_sym[peer]) { set_err("peer %d not mapped", peer); return -2; }
  TF_LAUNCH(launch_probe(X.peer_sym[peer], X.rank, value, (cudaStream_t)stream));
  return 0;
}

int tile_dist_probe_read(tf_dist_t h, int32_t* out) {
  if (!h) return -1;
  if (!out) return -2;
  DistRank& X = h->r;
  TF_CUDA(cudaDeviceSynchronize());
  TF_CUDA(cudaMemcpy(out, (char*)X.sym.p + SY_PROBE * sizeof(int), (TF_MAX_RANKS + 1) * sizeof(int),
                     cudaMemcpyDeviceToHost));
  return 0;
}

void tile_dist_close(tf_dist_t h) {
  if (!h) return;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  g_handles.erase(&h->r);
  dist_destroy(h->r);
  delete h;
}

int tile_dist_emulate(int alg, int64_t n, int64_t b, int64_t ib, int P, int Q, double* const* dA_loc,
                      double* const* dAux_loc, int32_t* const* dIpiv_loc, int32_t* d_info, tf_stream_t stream) {
  int rc = check_dist_args(alg, n, b, ib, P, Q);
  if (rc) return rc;
  if (!dA_loc) return -7;
  if (alg != 0 && !dAux_loc) return -8;
  if (alg == 2 && !dIpiv_loc) return -9;
  if (!d_info) return -10;
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  int dev;
  TF_CUDA(cudaGetDevice(&dev));
  if ((rc = device_setup(dev))) return rc;
  const int R = P * Q;
  const int ctas = g_ctas > 0 ? std::min(g_ctas, g_nsm[dev]) : g_nsm[dev];  // all co-resident
  if (ctas < R) { set_err("need at least one CTA per emulated rank"); return TF_ERR_UNSUPPORTED; }
  EmuKey key{dev, alg, n, b, ib, P, Q, g_policy};
  auto& ranks = g_emu[key];
  if (ranks.empty()) {
    for (int r = 0; r < R; ++r) {
      ranks.emplace_back(new DistRank());
      if ((rc = dist_create(*ranks.back(), alg, n, b, ib, P, Q, r))) {
        for (auto& x : ranks) dist_destroy(*x);
        ranks.clear();
        g_emu.erase(key);
        return rc;
      }
    }
    for (int r = 0; r < R; ++r)
      for (int q = 0; q < R; ++q) ranks[r]->peer_sym[q] = (char*)ranks[q]->sym.p;
  }
  cudaStream_t s = (cudaStream_t)stream;
  static Runs RUN;
  memset(&RUN, 0, sizeof(RUN));
  RUN.nruns = R;
  for (int r = 0; r < R; ++r) {
    const int c0 = (int)((int64_t)r * ctas / R), c1 = (int)((int64_t)(r + 1) * ctas / R);
    // only rank 0 writes the caller's d_info (all ranks compute the same combined value)
    if ((rc = dist_prepare(*ranks[r], RUN.r[r], c0, c1 - c0, dA_loc[r], dAux_loc ? dAux_loc[r] : nullptr,
                           dIpiv_loc ? dIpiv_loc[r] : nullptr, r == 0 ? d_info : nullptr, s)))
      return rc;
  }
  TF_LAUNCH(launch_persistent(RUN, ctas, smem_bytes(), s, true));
  return 0;
}

// ---------------------------------------------------------------- errors, teardown
const char* tile_strerror(int code) {
  switch (code) {
    case 0: return "success";
    case TF_ERR_CUDA: return "CUDA runtime error";
    case TF_ERR_NOMEM: return "device allocation failed";
    case TF_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return code < 0 ? "invalid argument" : "unknown error";
  }
}

const char* tile_last_error(void) { return g_err; }

void tile_finalize(void) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  for (auto& kv : g_ws) {
    Workspace& W = kv.second;
    for (Buf* b : {&W.state, &W.q, &W.vx, &W.scratch, &W.info, &W.trace, &W.xt, &W.hostA, &W.hostAux, &W.hostPiv,
                   &W.flags})
      release(*b);
  }
  g_ws.clear();
  for (auto& kv : g_dags) free_dag(kv.second);
  g_dags.clear();
  for (auto& kv : g_emu)
    for (auto& x : kv.second) dist_destroy(*x);
  g_emu.clear();
  g_plans.clear();
  g_last_ws = nullptr;
  for (int d = 0; d < 64; ++d) g_attr_set[d] = false;
}

}  // extern "C"
