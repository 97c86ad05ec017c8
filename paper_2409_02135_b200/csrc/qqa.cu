// qqa.cu -- host engine and C ABI of libqqa.so (declared in include/qqa.h).
//
// One handle = one GPU's shard of the replica ensemble. Per annealing step the
// engine launches ONE fused kernel (k_step) on the caller's stream; with a
// communicator attached it follows it with one ncclAllReduce of the 2n int64
// replica-statistic sums (the only cross-GPU exchange of the method, Eq. 10).
#include "qqa.h"
#include "qqa_dispatch.h"

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // NVTX ranges (header-only v3): create / run / evaluate in nsys / ncu timelines

#include <algorithm>
#include <cmath>
#include <memory>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;

// RAII NVTX range around an entry point (SURVEY.md §5 tracing).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

#define QQA_CUDA(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(QQA_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define QQA_NCCL(call)                                                                      \
  do {                                                                                      \
    ncclResult_t r_ = (call);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return fail(QQA_ERR_COMM, std::string(#call) + ": " + ncclGetErrorString(r_));        \
  } while (0)

constexpr size_t kAlign = 256;
constexpr int kSchedCap = 4096;   // steps per persistent launch (device table of per-step scalars)
constexpr int64_t kClusterMaxElems = 1 << 15;   // n S_p up to this runs in one thread-block cluster (k_run_cluster)
constexpr int64_t kClusterMaxGather = 1 << 19;  // ... if its DSMEM gather (padded nnz x S_p values per step) is small
constexpr double kL2BlockBudget = 128.0 * 1024 * 1024;  // p larger than this is replica-blocked (measured)
constexpr double kKaryChunkBudget = 32.0 * 1024 * 1024; // K-ary: gathered lines of one replica chunk (measured, §4)
size_t up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Shape {
  int n = 0;
  int64_t nnz = 0;   // of the graph the kernels walk (complement for max clique)
  int S_local = 0, S_total = 0;
  int SB = 0, B = 0, S_p = 0;  // replica blocks: S_p = B * SB local columns, layout [B][n+1][SB]
  int W = 0, lanes = 0, vpl = 0;
  int64_t nnz_pad = 0;         // row-padded CSR (rows rounded up to 4 entries)
  int G = 1;                   // instances of a batch (NEXT-3); 1 without group_of_row
  bool kary = false;           // graph colouring (NEXT-4): layout [n][S_local][KP]
  bool weighted = false;       // edge weights (MIS / Max-Cut)
  int K = 0, KP = 0, LK = 0;   // colours, padded to a multiple of 4, lanes per variable
  int KS = 1;                  // source segments of the segmented gather; 1: one-pass k_step
  int64_t nnz_seg = 0;         // entries of the segment CSRs (each (row, segment) padded to 4)
};

struct Layout {
  size_t rowptr, colidx, rowptr_pad, colidx_pad, gor, theta, m, v, p0, p1, c0, c1, ms, s0, s1, s2, flag, X,
      counts, tot, energy, best, beste, genergy, gbest, gbeste, xbuf, sched, cs0, cs1, w, w_pad, wdeg, wsums,
      rowptr_seg, colidx_seg, total;
};

Layout make_layout(const Shape& s) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = up(o + std::max<size_t>(bytes, 1), kAlign); return at; };
  const size_t ns = s.kary ? (size_t)s.n * s.S_local * s.KP * sizeof(float)
                           : ((size_t)s.n + 1) * s.S_p * sizeof(float);
  const size_t nk = (size_t)s.n * (s.kary ? s.K : 1);   // statistics entries: per (variable[, colour])
  L.rowptr = take(((size_t)s.n + 1) * sizeof(int));
  L.colidx = take((size_t)s.nnz * sizeof(int));
  L.rowptr_pad = take(((size_t)s.n + 1) * sizeof(int));
  L.colidx_pad = take((size_t)s.nnz_pad * sizeof(int));
  L.gor = take((size_t)s.n * sizeof(int));
  L.theta = take(s.kary ? 0 : ns);   // K-ary: the parameter is P itself (p0 / p1)
  L.m = take(ns);
  L.v = take(ns);
  L.p0 = take(ns);
  L.p1 = take(ns);
  L.c0 = take(nk * sizeof(float));
  L.c1 = take(nk * sizeof(float));
  L.ms = take(nk * sizeof(float2));
  L.s0 = take(2 * nk * sizeof(long long));
  L.s1 = take(2 * nk * sizeof(long long));
  L.s2 = take(2 * nk * sizeof(long long));
  L.flag = take(4 * sizeof(int));
  L.X = take(s.kary ? (size_t)s.n * s.S_local : (size_t)s.n * s.W * sizeof(uint32_t));   // K-ary: uint8 colours
  L.counts = take(3 * (size_t)s.S_total * s.G * sizeof(long long));   // [S_total][G][3]
  L.tot = take(3 * (size_t)s.S_total * sizeof(long long));            // [S_total][3] summed over instances
  L.energy = take((size_t)s.S_total * sizeof(double));
  L.best = take(sizeof(int));
  L.beste = take(sizeof(double));
  L.genergy = take((size_t)s.S_total * s.G * sizeof(double));         // [G][S_total]
  L.gbest = take((size_t)s.G * sizeof(int));
  L.gbeste = take((size_t)s.G * sizeof(double));
  L.xbuf = take((size_t)s.n);
  L.sched = take((size_t)kSchedCap * sizeof(float4));
  L.cs0 = take((size_t)s.S_p * sizeof(long long));   // printed clique: column sums of p[0] / p[1]
  L.cs1 = take((size_t)s.S_p * sizeof(long long));
  L.w = take(s.weighted ? (size_t)s.nnz * sizeof(float) : 0);           // edge weights
  L.w_pad = take(s.weighted ? (size_t)s.nnz_pad * sizeof(float) : 0);   // aligned with colidx_pad
  L.wdeg = take(s.weighted ? (size_t)s.n * sizeof(float) : 0);
  L.wsums = take(2 * (size_t)s.S_total * sizeof(long long));            // [S_total][2] weight sums
  L.rowptr_seg = take(s.KS > 1 ? (size_t)s.KS * ((size_t)s.n + 1) * sizeof(int) : 0);   // [KS][n+1]
  L.colidx_seg = take(s.KS > 1 ? (size_t)s.nnz_seg * sizeof(int) : 0);
  L.total = o;
  return L;
}

int next_pow2(int x) { int p = 1; while (p < x) p <<= 1; return p; }

// Every lane of a step-kernel group holds a vector of the replica block (k_step / k_run FULL variant).
bool full_lanes(const Shape& s) { return s.SB / 8 == s.lanes * s.vpl; }

int check_config(const qqa_config* c) {
  if (!c) return fail(QQA_ERR_INVALID_ARG, "config is NULL");
  if (c->problem < 0 || c->problem > 4)
    return fail(QQA_ERR_INVALID_ARG,
                "problem must be 0 (MIS), 1 (Max-Cut), 2 (max clique), 3 (colouring) or 4 (max clique, sparse)");
  if (c->problem == QQA_COLORING && (c->n_colors < 2 || c->n_colors > 16))
    return fail(QQA_ERR_INVALID_ARG, "n_colors must be in 2..16 for QQA_COLORING");
  if (c->alpha < 2 || c->alpha > 16 || (c->alpha & 1)) return fail(QQA_ERR_INVALID_ARG, "alpha must be even, 2..16 (Eq. 7)");
  if (c->S_total < 1 || c->S_total > (1 << 20)) return fail(QQA_ERR_INVALID_ARG, "S_total must be in 1..2^20");
  if (c->S_local < 1) return fail(QQA_ERR_INVALID_ARG, "S_local must be >= 1");
  if (c->S_local > 1024) return fail(QQA_ERR_UNSUPPORTED, "S_local > 1024 replicas per GPU is not supported by this build");
  if (c->replica_offset < 0 || (int64_t)c->replica_offset + c->S_local > c->S_total)
    return fail(QQA_ERR_INVALID_ARG, "replica shard [offset, offset+S_local) must lie in [0, S_total)");
  if (!std::isfinite(c->lr) || !std::isfinite(c->penalty) || !std::isfinite(c->comm) || c->comm < 0.0f ||
      !(c->beta1 >= 0.0f && c->beta1 < 1.0f) || !(c->beta2 >= 0.0f && c->beta2 < 1.0f) || !(c->eps >= 0.0f) ||
      !std::isfinite(c->weight_decay) || !std::isfinite(c->init_lo) || !std::isfinite(c->init_hi))
    return fail(QQA_ERR_INVALID_ARG, "hyper-parameter out of range (lr, penalty, comm>=0, 0<=beta<1, eps>=0 ...)");
  if (c->map != QQA_MAP_SIGMOID && c->map != QQA_MAP_CLAMP)
    return fail(QQA_ERR_INVALID_ARG, "map must be 0 (sigmoid) or 1 (clamp)");
  if (!(c->temperature >= 0.0f) || !std::isfinite(c->temperature))
    return fail(QQA_ERR_INVALID_ARG, "temperature must be finite and >= 0");
  if (c->kary_grad != 0 && c->kary_grad != 1) return fail(QQA_ERR_INVALID_ARG, "kary_grad must be 0 or 1");
  return QQA_OK;
}

int check_graph(const qqa_graph* g) {
  if (!g) return fail(QQA_ERR_INVALID_ARG, "graph is NULL");
  if (g->n < 0 || g->nnz < 0) return fail(QQA_ERR_INVALID_ARG, "negative n or nnz");
  if (g->n > 0 && !g->rowptr) return fail(QQA_ERR_INVALID_ARG, "rowptr is NULL");
  if (g->nnz > 0 && !g->colidx) return fail(QQA_ERR_INVALID_ARG, "colidx is NULL");
  if (g->nnz >= (int64_t)INT32_MAX) return fail(QQA_ERR_UNSUPPORTED, "nnz >= 2^31 not supported by this build");
  if (g->n == 0) return QQA_OK;
  if (g->rowptr[0] != 0 || g->rowptr[g->n] != g->nnz) return fail(QQA_ERR_BAD_GRAPH, "rowptr[0] != 0 or rowptr[n] != nnz");
  for (int i = 0; i < g->n; ++i)
    if (g->rowptr[i + 1] < g->rowptr[i]) return fail(QQA_ERR_BAD_GRAPH, "rowptr is not non-decreasing");
  if (g->group_of_row) {  // batch of instances (NEXT-3): contiguous row ranges 0..n_groups-1
    if (g->n_groups < 1 || g->n_groups > (1 << 24)) return fail(QQA_ERR_INVALID_ARG, "n_groups must be in 1..2^24");
    for (int i = 0; i < g->n; ++i) {
      const int k = g->group_of_row[i];
      if (k < 0 || k >= g->n_groups) return fail(QQA_ERR_BAD_GRAPH, "group_of_row out of [0, n_groups)");
      if (i > 0 && k < g->group_of_row[i - 1])
        return fail(QQA_ERR_BAD_GRAPH, "group_of_row must be non-decreasing (instances are contiguous row ranges)");
    }
  }
  return QQA_OK;
}

// Row range [a, b) of the instance holding row i (the whole graph without groups).
void instance_range(const qqa_graph* g, int i, int& a, int& b) {
  if (!g->group_of_row) { a = 0; b = g->n; return; }
  const int k = g->group_of_row[i];
  a = i; b = i + 1;
  while (a > 0 && g->group_of_row[a - 1] == k) --a;
  while (b < g->n && g->group_of_row[b] == k) ++b;
}

int64_t problem_nnz(const qqa_graph* g, int problem) {
  if (problem != QQA_MAXCLIQUE) return g->nnz;
  if (!g->group_of_row) return (int64_t)g->n * (g->n - 1) - g->nnz;
  int64_t pairs = 0;  // sum over instances of n_k (n_k - 1)
  for (int i = 0; i < g->n;) {
    int a, b;
    instance_range(g, i, a, b);
    pairs += (int64_t)(b - a) * (b - a - 1);
    i = b;
  }
  return pairs - g->nnz;
}

// Segmented gather: segment k of the sources is [seg_lo(n, KS, k), seg_lo(n, KS, k + 1)).
int seg_lo(int n, int KS, int k) { return (int)((int64_t)n * k / KS); }

// Segment CSR: for every segment k, row i's neighbours in segment k (CSR order), padded to a multiple of 4
// with the sentinel n. rp: [KS][n+1] absolute offsets into ci. Returns the entry count; fills rp / ci if given.
// One pass over each row (its columns ascend, so the segment index only moves forward): O(nnz + KS n).
int64_t build_seg_csr(const int64_t* rowptr, const int32_t* colidx, int n, int KS, int* rp, int* ci) {
  std::vector<int> lo((size_t)KS + 1);
  for (int k = 0; k <= KS; ++k) lo[k] = seg_lo(n, KS, k);
  if (const char* env = std::getenv("QQA_SEG_SPLIT")) {   // experiment: every source in segment 0, the last
    if (std::atoi(env) != 0)                              // pass an update without a gather
      for (int k = 1; k < KS; ++k) lo[k] = n;
  }
  lo[KS] = INT32_MAX;   // the last segment takes everything from lo[KS-1] on (incl. out-of-range columns)
  std::vector<int> cnt(rp ? (size_t)KS * n : 0);
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {   // segment boundaries of a row by binary search (its columns ascend)
    const int32_t* a = colidx + rowptr[i];
    const int32_t* end = colidx + rowptr[i + 1];
    for (int k = 0; k < KS; ++k) {
      const int32_t* b = (k + 1 < KS) ? std::lower_bound(a, end, lo[k + 1]) : end;
      const int c = (int)(b - a);
      total += (c + 3) / 4 * 4;
      if (rp) cnt[(size_t)k * n + i] = c;
      a = b;
    }
  }
  if (!rp) return total;
  int64_t o = 0;
  for (int k = 0; k < KS; ++k) {
    for (int i = 0; i < n; ++i) {
      rp[(size_t)k * (n + 1) + i] = (int)o;
      o += (cnt[(size_t)k * n + i] + 3) / 4 * 4;
    }
    rp[(size_t)k * (n + 1) + n] = (int)o;
  }
  if (ci) {
    for (int i = 0; i < n; ++i) {
      int64_t e = rowptr[i];
      for (int k = 0; k < KS; ++k) {
        int o2 = rp[(size_t)k * (n + 1) + i];
        const int c = cnt[(size_t)k * n + i];
        for (int q = 0; q < c; ++q) ci[o2++] = colidx[e++];
        for (int q = c; q < (c + 3) / 4 * 4; ++q) ci[o2++] = n;
      }
    }
  }
  return o;
}

int make_shape(const qqa_graph* g, const qqa_config* c, Shape& s) {
  int st = check_graph(g);
  if (st) return st;
  if ((st = check_config(c))) return st;
  if (c->problem == QQA_MAXCLIQUE && g->n > 65536) return fail(QQA_ERR_UNSUPPORTED, "max clique: n > 65536 (dense complement)");
  s.n = g->n;
  s.nnz = problem_nnz(g, c->problem);
  if (s.nnz >= (int64_t)INT32_MAX) return fail(QQA_ERR_UNSUPPORTED, "complement nnz >= 2^31");
  s.S_local = c->S_local;
  s.S_total = c->S_total;
  s.G = g->group_of_row ? g->n_groups : 1;
  if (g->weights) {
    if (c->problem != QQA_MIS && c->problem != QQA_MAXCUT)
      return fail(QQA_ERR_UNSUPPORTED, "edge weights are supported for MIS and Max-Cut (P:687)");
    if (g->group_of_row) return fail(QQA_ERR_UNSUPPORTED, "batches (group_of_row) of weighted graphs are not supported");
    s.weighted = true;
  }
  if (c->problem == QQA_MAXCLIQUE_SPARSE && g->group_of_row)
    return fail(QQA_ERR_UNSUPPORTED, "batches (group_of_row) are not supported for the sparse max-clique relaxation");
  if (c->problem == QQA_COLORING) {
    if (g->group_of_row) return fail(QQA_ERR_UNSUPPORTED, "batches (group_of_row) are not supported for colouring");
    s.kary = true;
    s.K = c->n_colors;
    s.KP = (s.K + 3) / 4 * 4;
    s.LK = std::max(4, std::min(32, next_pow2(c->S_local)));
    // The step walks (replica chunk, variable) items chunk-major, so while the grid sweeps a chunk only
    // that chunk's lines of P are gathered: n LK KP 4 bytes. Chunks are narrowed until that fits the
    // ~32 MB an all-SM gather keeps in L2 (k8: 32 -> 8 lanes, 836 -> 706 us per step).
    while (s.LK > 4 && (double)g->n * s.LK * s.KP * sizeof(float) > kKaryChunkBudget) s.LK >>= 1;
    if (const char* env = std::getenv("QQA_KARY_LANES")) s.LK = std::max(4, std::min(32, next_pow2(std::atoi(env))));
  }
  // Replica blocking: when one copy of p is larger than the L2
  // budget, split the replicas into blocks of SB (a power of two >= 8) so that
  // one block of p -- the gathered working set while the grid sweeps it -- fits.
  const int S8 = (c->S_local + 7) / 8 * 8;
  const double p_bytes = (double)s.n * S8 * sizeof(float);
  int SB = S8;
  const char* env = std::getenv("QQA_BLOCK_REPLICAS");
  if (s.kary) {
    SB = S8;  // no replica blocking in the K-ary layout
  } else if (env && std::atoi(env) > 0) {
    SB = std::max(8, next_pow2(std::atoi(env)));
  } else if (p_bytes > kL2BlockBudget && s.n > 0) {
    SB = 8;
    while (SB * 2 < S8 && (double)s.n * (SB * 2) * sizeof(float) <= kL2BlockBudget) SB *= 2;
  }
  if (SB >= S8) SB = S8;
  s.SB = SB;
  s.B = (S8 + SB - 1) / SB;
  s.S_p = s.B * SB;
  s.W = (c->S_local + 31) / 32;
  const int SB8 = SB / 8;  // 8-replica vectors (one 256-bit access) per item
  s.lanes = std::min(32, next_pow2(SB8));
  s.vpl = next_pow2((SB8 + s.lanes - 1) / s.lanes);
  s.nnz_pad = 0;
  for (int i = 0; i < s.n; ++i) {
    int a = 0, b = s.n;
    if (c->problem == QQA_MAXCLIQUE) instance_range(g, i, a, b);
    const int64_t deg = (c->problem == QQA_MAXCLIQUE) ? (int64_t)(b - a - 1) - (g->rowptr[i + 1] - g->rowptr[i])
                                                      : g->rowptr[i + 1] - g->rowptr[i];
    s.nnz_pad += (deg + 3) / 4 * 4;
  }
  if (s.nnz_pad >= (int64_t)INT32_MAX) return fail(QQA_ERR_UNSUPPORTED, "padded nnz >= 2^31");
  // Segmented gather: VPL 1, FULL shapes, unweighted, MIS / Max-Cut on the given graph.
  s.KS = 1;
  if (const char* env = std::getenv("QQA_SEGMENTS")) s.KS = std::max(1, std::min(64, std::atoi(env)));
  if (s.KS > 1 && (s.kary || s.weighted || s.vpl != 1 || !full_lanes(s) || s.n < 4 * s.KS ||
                   (c->problem != QQA_MIS && c->problem != QQA_MAXCUT)))
    s.KS = 1;
  if (s.KS > 1) {
    s.nnz_seg = build_seg_csr(g->rowptr, g->colidx, s.n, s.KS, nullptr, nullptr);
    if (s.nnz_seg >= (int64_t)INT32_MAX) s.KS = 1;
  }
  if ((int64_t)s.B * ((int64_t)s.n + 1) * s.SB >= (int64_t)1 << 40) return fail(QQA_ERR_UNSUPPORTED, "state too large");
  return QQA_OK;
}

// Host check of the ORIGINAL CSR for QQA_MAXCLIQUE (the device k_validate runs on the graph the
// kernels walk, which for the dense clique is the complement; the complement is built from the
// original on the host, so the original must be checked before it is indexed). Same conditions as
// k_validate: columns in [0, n), rows strictly ascending (no duplicates), no self-loops, symmetric,
// no edge between two instances of a batch.
int validate_host(const qqa_graph* g) {
  const int n = g->n;
  for (int i = 0; i < n; ++i) {
    int64_t prev = -1;
    for (int64_t e = g->rowptr[i]; e < g->rowptr[i + 1]; ++e) {
      const int j = g->colidx[e];
      if (j < 0 || j >= n) return fail(QQA_ERR_BAD_GRAPH, "graph rejected: column out of range;");
      if (j <= prev) return fail(QQA_ERR_BAD_GRAPH, "graph rejected: row not strictly ascending (unsorted or duplicate);");
      if (j == i) return fail(QQA_ERR_BAD_GRAPH, "graph rejected: self-loop;");
      if (g->group_of_row && g->group_of_row[j] != g->group_of_row[i])
        return fail(QQA_ERR_BAD_GRAPH, "graph rejected: edge between two instances of the batch;");
      prev = j;
    }
  }
  for (int i = 0; i < n; ++i)   // symmetry (rows are sorted now): i must appear in row j
    for (int64_t e = g->rowptr[i]; e < g->rowptr[i + 1]; ++e) {
      const int j = g->colidx[e];
      const int32_t* a = g->colidx + g->rowptr[j];
      const int32_t* b = g->colidx + g->rowptr[j + 1];
      const int32_t* f = std::lower_bound(a, b, i);
      if (f == b || *f != i) return fail(QQA_ERR_BAD_GRAPH, "graph rejected: not symmetric;");
    }
  return QQA_OK;
}

// Complement CSR (max clique = MIS on the complement graph); for a batch
// the complement is taken inside each instance (block-diagonal union of complements).
void build_complement(const qqa_graph* g, std::vector<int>& rp, std::vector<int>& ci) {
  const int n = g->n;
  rp.assign((size_t)n + 1, 0);
  ci.clear();
  ci.reserve((size_t)problem_nnz(g, QQA_MAXCLIQUE));
  std::vector<char> mark((size_t)n, 0);
  for (int i = 0; i < n; ++i) {
    int a, b;
    instance_range(g, i, a, b);
    for (int64_t e = g->rowptr[i]; e < g->rowptr[i + 1]; ++e) mark[g->colidx[e]] = 1;
    for (int j = a; j < b; ++j)
      if (j != i && !mark[j]) ci.push_back(j);
    for (int64_t e = g->rowptr[i]; e < g->rowptr[i + 1]; ++e) mark[g->colidx[e]] = 0;
    rp[i + 1] = (int)ci.size();
  }
}

}  // namespace

struct qqa_handle {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  qqa_config cfg{};
  Shape s;
  Layout L{};
  char* ws = nullptr;
  int* rowptr = nullptr;
  int* colidx = nullptr;
  int* rowptr_pad = nullptr;
  int* colidx_pad = nullptr;
  float *theta = nullptr, *m = nullptr, *v = nullptr, *p[2] = {nullptr, nullptr}, *c[2] = {nullptr, nullptr};
  long long* sums[3] = {nullptr, nullptr, nullptr};
  float2* ms = nullptr;
  int* flag = nullptr;
  uint32_t* X = nullptr;
  int* gor = nullptr;          // group_of_row on the device (NULL without a batch)
  unsigned long long* counts = nullptr;
  long long* tot = nullptr;
  double* energy = nullptr;
  int* best = nullptr;
  double* beste = nullptr;
  double* genergy = nullptr;
  int* gbest = nullptr;
  double* gbeste = nullptr;
  uint8_t* xbuf = nullptr;
  float4* sched = nullptr;     // per-step scalars of a persistent launch
  long long* colsum[2] = {nullptr, nullptr};   // printed clique: per-replica column sums of p[0] / p[1]
  float* w = nullptr;          // edge weights (NULL unweighted), padded copy, weighted degrees
  float* w_pad = nullptr;
  float* wdeg = nullptr;
  long long* wsums = nullptr;  // [S_total][2] evaluation weight sums (fixed point 2^24)
  bool serpentine = false;     // replica blocks swept in alternating order step to step (QQA_SERPENTINE)
  qqa::StepKernel kst = nullptr;   // k_step_st (staged state) for the launch-per-step path, nullptr: k_step
  // segmented gather (s.KS > 1): segment CSRs and the three kernels (first / middle partial passes, last + update)
  int* rowptr_seg = nullptr;
  int* colidx_seg = nullptr;
  qqa::StepKernel kseg[3] = {nullptr, nullptr, nullptr};
  int grid_seg[3] = {0, 0, 0};
  int grid_st = 0;
  size_t st_smem = 0;
  int grid_run = 0;            // co-resident grid of k_run (0: launch-per-step only)
  int run_cta = 256;           // threads per CTA of k_run (1024: contiguous rows per SM)
  // fused statistics exchange over peer memory (qqa_attach_exchange; k_step_x instead of k_step + NCCL)
  bool xmode = false;
  int xrank = 0, xG = 1;
  long long* xsums[qqa::kMaxRanks][3] = {};     // every rank's sums buffers, mapped in this process
  unsigned long long* xflag[qqa::kMaxRanks] = {};
  unsigned int* xticket = nullptr;
  unsigned long long xsync = 0;                  // barriers so far (each adds G arrivals to every counter)
  bool xslotted = false;                         // owner-slotted exchange (k_step_xs) instead of atomics
  bool xdefer_init = false;                      // slotted, no communicator: qqa_loopback_sync_init scatters
  long long* xbase[qqa::kMaxRanks] = {};         // every rank's exchange buffer (slots, then totals)
  int grid_xs = 0;                               // co-resident grid of k_step_xs (cooperative launch)
  long long* ws_sums[3] = {nullptr, nullptr, nullptr};   // the workspace's own sums (get_stats scratch)
  int cluster_cs = 0;          // k_run_cluster: CTAs per cluster (0: not available for this handle)
  qqa::StepKKernel kq = nullptr;    // K-ary colour-quad step (KP 12 / 16), nullptr: k_step_K
  int grid_kq = 0;
  int cluster_rows = 0;        // rows per CTA of the cluster
  size_t cluster_smem = 0;
  int cur = 0;   // p / c buffer of the current step (mod 2)
  int scur = 0;  // sums buffer of the current step (mod 3)
  int64_t step = 0;
  ncclComm_t comm = nullptr;
  std::shared_ptr<ncclComm_t> comm_box;   // owner of comm (shared by qqa_share_comm; destroyed with the last user)
  int rank = 0, nranks = 1;
  int grid_step = 0, grid_init = 0, grid_fin = 0;
  // compute / all-reduce overlap (N > 1): the step's rows run as comm_chunks launches; chunk c's
  // sums are all-reduced on cstream while chunk c+1 computes
  int comm_chunks = 1;
  cudaStream_t cstream = nullptr;
  std::vector<cudaEvent_t> chunk_ev;   // [comm_chunks] chunk computed; [comm_chunks] all-reduces done
  bool profiling = false;
  std::vector<cudaEvent_t> ev;  // pairs (start, end)
  size_t ev_used = 0;
  int64_t prof_launches = 0;
  double prof_ms = 0.0;
  int64_t launches = 0;
};

namespace {

using StepKernel = qqa::StepKernel;
using InitKernel = void (*)(const qqa::InitParams);
using RunKernel = qqa::RunKernel;

// Step-kernel mode: bit 0 clamp map, bit 1 Langevin noise (template, so the
// default sigmoid / no-noise kernel carries none of the optional code).
int step_mode(const qqa_config& c, bool weighted = false) {
  return (c.map == QQA_MAP_CLAMP ? qqa::kModeClamp : 0) | (c.temperature > 0.0f ? qqa::kModeNoise : 0) |
         (c.problem == QQA_MAXCLIQUE_SPARSE ? qqa::kModeSparseClique : 0) | (weighted ? qqa::kModeWeighted : 0);
}

template <int L, int V>
InitKernel init_for() { return qqa::k_init<L, V>; }

// run_cta: 1024 (contiguous rows per SM) or 256 threads per CTA of the persistent kernel (VPL 1 only).
// The k_step / k_run instantiations live in k_mode<mode>.cu (compiled in parallel).
bool pick_kernels(int lanes, int vpl, int mode, StepKernel& ks, InitKernel& ki, RunKernel* kr = nullptr,
                  int run_cta = 256, bool full = false) {
  switch (mode) {
    case 0: ks = qqa::step_kernel_m0(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m0(lanes, vpl, run_cta, full); break;
    case 1: ks = qqa::step_kernel_m1(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m1(lanes, vpl, run_cta, full); break;
    case 2: ks = qqa::step_kernel_m2(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m2(lanes, vpl, run_cta, full); break;
    case 3: ks = qqa::step_kernel_m3(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m3(lanes, vpl, run_cta, full); break;
    case 4: ks = qqa::step_kernel_m4(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m4(lanes, vpl, run_cta, full); break;
    case 5: ks = qqa::step_kernel_m5(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m5(lanes, vpl, run_cta, full); break;
    case 6: ks = qqa::step_kernel_m6(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m6(lanes, vpl, run_cta, full); break;
    case 7: ks = qqa::step_kernel_m7(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m7(lanes, vpl, run_cta, full); break;
    case 8: ks = qqa::step_kernel_m8(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m8(lanes, vpl, run_cta, full); break;
    case 9: ks = qqa::step_kernel_m9(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m9(lanes, vpl, run_cta, full); break;
    case 10: ks = qqa::step_kernel_m10(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m10(lanes, vpl, run_cta, full); break;
    case 11: ks = qqa::step_kernel_m11(lanes, vpl, full); if (kr) *kr = qqa::run_kernel_m11(lanes, vpl, run_cta, full); break;
    default: ks = nullptr; if (kr) *kr = nullptr; break;
  }
  ki = nullptr;
#define QQA_ICASE(L, V) \
  if (lanes == L && vpl == V) ki = init_for<L, V>();
  QQA_ICASE(1, 1) QQA_ICASE(2, 1) QQA_ICASE(4, 1) QQA_ICASE(8, 1) QQA_ICASE(16, 1)
  QQA_ICASE(32, 1) QQA_ICASE(32, 2) QQA_ICASE(32, 4)
#undef QQA_ICASE
  return ks != nullptr && ki != nullptr;
}

uint64_t mix64_host(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------- K-ary kernels
using StepKKernel = qqa::StepKKernel;
using InitKKernel = qqa::InitKKernel;
using PackKKernel = qqa::PackKKernel;

bool pick_kary(int KP, int K, int mode, StepKKernel& ks, InitKKernel& ki, PackKKernel& kp) {
  return qqa::kary_kernels(KP, K, mode, ks, ki, kp);   // k_kary.cu
}

// k_t of the K-ary entropy: -gamma c_K alpha K, c_K = 1/((K-1)((K-1)^(alpha-1) + 1)) (host double -> fp32)
float kt_kary(int K, int alpha, float gamma) {
  const double cK = 1.0 / ((double)(K - 1) * (std::pow((double)(K - 1), (double)(alpha - 1)) + 1.0));
  return (float)(-(double)gamma * cK * (double)alpha * (double)K);
}

int grid_for(const void* kernel, int sm_count, int64_t items, int lanes, int& grid, int threads = 256) {
  int per_sm = 0;
  QQA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0));
  const int need = (int)std::max<int64_t>(1, std::min<int64_t>(INT32_MAX, (items * lanes + threads - 1) / threads));
  grid = std::max(1, std::min(need, std::max(1, per_sm) * sm_count));
  return QQA_OK;
}

// Printed clique relaxation: column sums of p[buf] into colsum[buf] (exact int64).
int launch_colsum(qqa_handle* h, int buf) {
  const Shape& s = h->s;
  QQA_CUDA(cudaMemsetAsync(h->colsum[buf], 0, (size_t)s.S_p * sizeof(long long), h->stream));
  if (s.n == 0) return QQA_OK;
  const int T = std::max(s.S_p, (h->sm_count * 4 * 256) / s.S_p * s.S_p);
  qqa::k_colsum<<<(T + 255) / 256, 256, 0, h->stream>>>(h->p[buf], s.n, s.SB, s.S_p, s.S_local, T,
                                                        (unsigned long long*)h->colsum[buf]);
  QQA_CUDA(cudaGetLastError());
  h->launches++;
  return QQA_OK;
}

int problem_kind(int problem) {   // the kernels' problem code (max clique = MIS on the complement)
  return problem == QQA_MAXCUT ? qqa::kMAXCUT : problem == QQA_MAXCLIQUE_SPARSE ? qqa::kMAXCLIQUE_SPARSE : qqa::kMIS;
}

int launch_init_kary(qqa_handle* h, bool use_given, const float* c_given) {
  const Shape& s = h->s;
  StepKKernel ks;
  InitKKernel ki;
  PackKKernel kp;
  pick_kary(s.KP, s.K, step_mode(h->cfg, h->s.weighted), ks, ki, kp);
  qqa::InitKParams P{};
  P.p0 = h->p[0]; P.p1 = h->p[1]; P.m = h->m; P.v = h->v;
  P.c = h->c[0]; P.sums = h->sums[0];
  P.n = s.n; P.S = s.S_local; P.K = s.K; P.S_total = s.S_total; P.replica_offset = h->cfg.replica_offset;
  P.base = mix64_host(h->cfg.seed);
  P.lo = (double)h->cfg.init_lo;
  P.hi = (double)h->cfg.init_hi;
  P.unif = (float)(1.0 / (double)s.K);
  P.use_given = use_given ? 1 : 0;
  P.c_given = c_given;
  const size_t nk = (size_t)s.n * s.K;
  for (int b = 0; b < 3; ++b) QQA_CUDA(cudaMemsetAsync(h->sums[b], 0, 2 * nk * sizeof(long long), h->stream));
  if (s.n > 0 && s.S_local > 0) {
    ki<<<h->grid_init, 256, 0, h->stream>>>(P);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  if (h->comm) QQA_NCCL(ncclAllReduce(h->sums[0], h->sums[0], 2 * nk, ncclInt64, ncclSum, h->comm, h->stream));
  h->cur = 0;
  h->scur = 0;
  QQA_CUDA(cudaMemsetAsync(h->flag, 0, 4 * sizeof(int), h->stream));
  return QQA_OK;
}

qqa::XParams make_xparams(const qqa_handle* h, int sa, int sb, int sz, int a, int b) {
  qqa::XParams X{};
  for (int r = 0; r < h->xG; ++r) {
    X.peer_cur[r] = h->xsums[r][sa];
    X.peer_next[r] = h->xsums[r][sb];
    X.peer_flag[r] = h->xflag[r];
  }
  X.zero = h->xsums[h->xrank][sz];
  X.flag = h->xflag[h->xrank];
  X.ticket = h->xticket;
  X.c_cur = h->c[a];
  X.c_next = h->c[b];
  X.ms = h->ms;
  X.expect = (unsigned long long)h->xG * h->xsync;
  X.rank = h->xrank;
  X.G = h->xG;
  X.rows_per_rank = std::max(1, (h->s.n + h->xG - 1) / h->xG);
  if (h->xslotted) {   // slots [2 parities][G][2][rpr] then totals [2][rpr] in every rank's buffer
    const size_t rpr = (size_t)X.rows_per_rank, G = (size_t)h->xG;
    const size_t pw = (size_t)((h->step + 1) & 1), pr = (size_t)(h->step & 1);   // step t = h->step + 1
    for (int r = 0; r < h->xG; ++r) {
      X.slot_w[r] = h->xbase[r] + ((pw * G + (size_t)h->xrank) * 2) * rpr;
      X.totals[r] = h->xbase[r] + 2 * G * 2 * rpr;
    }
    X.slot_r = h->xbase[h->xrank] + (pr * G) * 2 * rpr;
  }
  return X;
}

// Owner-slotted exchange: this rank's partial sums of the initial statistics (sums[0], not all-reduced)
// into its slot (parity 0) at every owner; the arrival that follows ends "step 0".
int xs_scatter_init(qqa_handle* h) {
  qqa::XParams X = make_xparams(h, h->scur, h->scur, h->scur, h->cur, h->cur);
  const size_t rpr = (size_t)X.rows_per_rank, G = (size_t)h->xG;
  for (int r = 0; r < h->xG; ++r) X.slot_w[r] = h->xbase[r] + ((0 * G + (size_t)h->xrank) * 2) * rpr;
  if (h->s.n > 0) {
    const int blocks = std::max(1, std::min((h->s.n + 255) / 256, h->sm_count * 8));
    qqa::k_xs_scatter<<<blocks, 256, 0, h->stream>>>(X, h->s.n, h->sums[0]);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  return QQA_OK;
}

// This rank's arrival at an exchange barrier (after the initial statistics are complete).
int x_arrive(qqa_handle* h) {
  const qqa::XParams X = make_xparams(h, h->scur, h->scur, h->scur, h->cur, h->cur);
  qqa::k_x_arrive<<<1, 32, 0, h->stream>>>(X);
  QQA_CUDA(cudaGetLastError());
  h->launches++;
  h->xsync++;
  return QQA_OK;
}

qqa::XStepKernel pick_xstep(int lanes, int vpl, int mode, bool full) {
  switch (mode) {
    case 0: return qqa::xstep_kernel_m0(lanes, vpl, full);
    case 1: return qqa::xstep_kernel_m1(lanes, vpl, full);
    case 2: return qqa::xstep_kernel_m2(lanes, vpl, full);
    case 3: return qqa::xstep_kernel_m3(lanes, vpl, full);
    case 8: return qqa::xstep_kernel_m8(lanes, vpl, full);
    case 9: return qqa::xstep_kernel_m9(lanes, vpl, full);
    case 10: return qqa::xstep_kernel_m10(lanes, vpl, full);
    case 11: return qqa::xstep_kernel_m11(lanes, vpl, full);
    default: return nullptr;
  }
}

qqa::XStepKernel pick_xsstep(int lanes, int vpl, int mode, bool full) {
  switch (mode) {
    case 0: return qqa::xsstep_kernel_m0(lanes, vpl, full);
    case 1: return qqa::xsstep_kernel_m1(lanes, vpl, full);
    case 2: return qqa::xsstep_kernel_m2(lanes, vpl, full);
    case 3: return qqa::xsstep_kernel_m3(lanes, vpl, full);
    case 8: return qqa::xsstep_kernel_m8(lanes, vpl, full);
    case 9: return qqa::xsstep_kernel_m9(lanes, vpl, full);
    case 10: return qqa::xsstep_kernel_m10(lanes, vpl, full);
    case 11: return qqa::xsstep_kernel_m11(lanes, vpl, full);
    default: return nullptr;
  }
}

int launch_init(qqa_handle* h, bool use_given, const float* c_given) {
  if (h->s.kary) return launch_init_kary(h, use_given, c_given);
  StepKernel ks;
  InitKernel ki;
  pick_kernels(h->s.lanes, h->s.vpl, step_mode(h->cfg, h->s.weighted), ks, ki);
  qqa::InitParams P{};
  P.theta = h->theta; P.m = h->m; P.v = h->v; P.p0 = h->p[0]; P.p1 = h->p[1];
  P.c = h->c[0]; P.sums = h->sums[0];
  P.n = h->s.n; P.SB = h->s.SB; P.B = h->s.B; P.S_local = h->s.S_local; P.S_total = h->s.S_total;
  P.replica_offset = h->cfg.replica_offset;
  P.base = mix64_host(h->cfg.seed);  // base = mix64(seed), computed on the host with the same mixer
  P.clamp = h->cfg.map == QQA_MAP_CLAMP ? 1 : 0;
  P.lo = (double)h->cfg.init_lo;
  P.hi = (double)h->cfg.init_hi;
  P.use_given = use_given ? 1 : 0;
  P.c_given = c_given;
  QQA_CUDA(cudaMemsetAsync(h->sums[0], 0, 2 * (size_t)h->s.n * sizeof(long long), h->stream));
  QQA_CUDA(cudaMemsetAsync(h->sums[1], 0, 2 * (size_t)h->s.n * sizeof(long long), h->stream));
  QQA_CUDA(cudaMemsetAsync(h->sums[2], 0, 2 * (size_t)h->s.n * sizeof(long long), h->stream));
  if (h->s.n > 0) {
    ki<<<h->grid_init, 256, 0, h->stream>>>(P);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  if (h->comm && !h->xslotted) {
    QQA_NCCL(ncclAllReduce(h->sums[0], h->sums[0], 2 * (size_t)h->s.n, ncclInt64, ncclSum, h->comm, h->stream));
  }
  h->cur = 0;
  h->scur = 0;
  if (h->xslotted && !h->xdefer_init) {   // slotted: partials to the owners' slots, then the first barrier
    int st;
    if ((st = xs_scatter_init(h))) return st;
    if ((st = x_arrive(h))) return st;
  } else if (h->xmode && h->comm && !h->xslotted) {   // every rank's sums[0] holds the totals: first barrier
    int st;
    if ((st = x_arrive(h))) return st;
  }
  if (h->cfg.problem == QQA_MAXCLIQUE_SPARSE) {
    int st;
    if ((st = launch_colsum(h, 0))) return st;
  }
  h->cur = 0;
  h->scur = 0;
  QQA_CUDA(cudaMemsetAsync(h->flag, 0, 4 * sizeof(int), h->stream));
  return QQA_OK;
}

int record_start(qqa_handle* h) {
  if (!h->profiling) return QQA_OK;
  if (h->ev_used + 2 > h->ev.size()) {
    for (int e = 0; e < 256; ++e) {
      cudaEvent_t x;
      QQA_CUDA(cudaEventCreate(&x));
      h->ev.push_back(x);
    }
  }
  QQA_CUDA(cudaEventRecord(h->ev[h->ev_used], h->stream));
  return QQA_OK;
}

int record_end(qqa_handle* h) {
  if (!h->profiling) return QQA_OK;
  QQA_CUDA(cudaEventRecord(h->ev[h->ev_used + 1], h->stream));
  h->ev_used += 2;
  h->prof_launches++;
  return QQA_OK;
}

// K-ary step loop: k_finalize over the n K (variable, colour) statistics, then k_step_K.
int do_steps_kary(qqa_handle* h, const float* gamma, int64_t n_steps) {
  const Shape& s = h->s;
  const qqa_config& c = h->cfg;
  StepKKernel ks;
  InitKKernel ki;
  PackKKernel kp;
  pick_kary(s.KP, s.K, step_mode(c, s.weighted), ks, ki, kp);
  const size_t nk = (size_t)s.n * s.K;
  qqa::StepKParams P{};
  P.rowptr = h->rowptr; P.colidx = h->colidx; P.m = h->m; P.v = h->v; P.flag = h->flag;
  P.n = s.n; P.S = s.S_local; P.K = s.K; P.L = s.LK;
  P.cmaj = 1;   // chunk-major item order (measured: k8 -4 % at the same chunk width, q13 -16 %)
  if (const char* env = std::getenv("QQA_KARY_CMAJ")) P.cmaj = std::atoi(env) != 0;
  P.Kf = (float)s.K; P.comm = c.comm; P.alpha = c.alpha;
  P.kgrad = c.kary_grad;
  P.b1 = c.beta1; P.c1 = (float)(1.0 - (double)c.beta1);
  P.b2 = c.beta2; P.c2 = (float)(1.0 - (double)c.beta2);
  P.eps = c.eps;
  P.unif = (float)(1.0 / (double)s.K);
  P.ns = (float)std::sqrt(2.0 * (double)c.lr * (double)c.temperature);
  P.S_total_u = (unsigned long long)s.S_total;
  const uint64_t nbase = mix64_host(c.seed ^ 0x6A09E667F3BCC909ull);
  for (int64_t k = 0; k < n_steps; ++k) {
    const int64_t t = h->step + 1;
    // xi key of (t, i, k, global s) = nbase + ((t n + i) K + k) S_total + s
    P.nkey = nbase + (uint64_t)t * (uint64_t)s.n * (uint64_t)s.K * (uint64_t)s.S_total + (uint64_t)c.replica_offset;
    P.kt = kt_kary(s.K, c.alpha, gamma[k]);
    P.at = (float)(1.0 - (double)c.lr * (double)c.weight_decay);
    P.st = (float)((double)c.lr / (1.0 - std::pow((double)c.beta1, (double)t)));
    P.rt = (float)(1.0 / std::sqrt(1.0 - std::pow((double)c.beta2, (double)t)));
    const int a = h->cur, b = h->cur ^ 1;
    const int sa = h->scur, sb = (h->scur + 1) % 3, sz = (h->scur + 2) % 3;
    P.p_cur = h->p[a]; P.p_next = h->p[b];
    P.ms = h->ms;
    P.sums_next = h->sums[sb];
    P.sums_zero = h->sums[sz];
    if (s.n > 0) {
      qqa::k_finalize_kc<<<h->grid_fin, 256, 0, h->stream>>>(h->c[a], h->sums[sa], (int)nk, (double)s.S_total,
                                                              c.comm, h->ms, h->c[b]);
      QQA_CUDA(cudaGetLastError());
      h->launches++;
      int st;
      if ((st = record_start(h))) return st;
      if (h->kq)
        h->kq<<<h->grid_kq, 256, 0, h->stream>>>(P);
      else
        ks<<<h->grid_step, 256, 0, h->stream>>>(P);
      QQA_CUDA(cudaGetLastError());
      h->launches++;
      if ((st = record_end(h))) return st;
    }
    if (h->comm) QQA_NCCL(ncclAllReduce(h->sums[sb], h->sums[sb], 2 * nk, ncclInt64, ncclSum, h->comm, h->stream));
    h->cur = b;
    h->scur = sb;
    h->step = t;
  }
  return QQA_OK;
}

int do_steps(qqa_handle* h, const float* gamma, int64_t n_steps);

// Persistent path (k_run): one cooperative launch per chunk of <= kSchedCap steps. Used for
// one-GPU, unblocked problems of up to 2^24 replica-variables (L2-resident / launch-bound);
// QQA_PERSISTENT=0/1 overrides. Bit-identical to the launch-per-step path.
bool use_persistent(const qqa_handle* h, int64_t n_steps) {
  if (h->grid_run <= 0 || h->comm || h->xmode || h->s.B != 1 || h->s.kary || h->s.n == 0 || n_steps < 2 ||
      h->cfg.problem == QQA_MAXCLIQUE_SPARSE)   // its column sums need a pass between steps
    return false;
  if (const char* env = std::getenv("QQA_PERSISTENT")) return std::atoi(env) != 0;
  return (int64_t)h->s.n * h->s.S_p <= ((int64_t)1 << 24);
}

int do_steps_persistent(qqa_handle* h, const float* gamma, int64_t n_steps) {
  StepKernel ks;
  InitKernel ki;
  RunKernel kr = nullptr;
  pick_kernels(h->s.lanes, h->s.vpl, step_mode(h->cfg, h->s.weighted), ks, ki, &kr, h->run_cta, full_lanes(h->s));
  const qqa_config& c = h->cfg;
  qqa::RunParams R{};
  qqa::StepParams& P = R.P;
  P.rowptr = h->rowptr; P.rowptr_pad = h->rowptr_pad; P.colidx_pad = h->colidx_pad;
  P.w_pad = h->w_pad; P.wdeg = h->wdeg;
  P.theta = h->theta; P.m = h->m; P.v = h->v; P.flag = h->flag;
  P.n = h->s.n; P.SB = h->s.SB; P.B = h->s.B; P.S_local = h->s.S_local; P.S_total = (double)h->s.S_total;
  P.row_begin = 0; P.row_end = h->s.n;
  P.problem = problem_kind(c.problem);
  P.alpha = c.alpha; P.lam = c.penalty; P.comm = c.comm;
  P.b1 = c.beta1; P.c1 = (float)(1.0 - (double)c.beta1);
  P.b2 = c.beta2; P.c2 = (float)(1.0 - (double)c.beta2);
  P.eps = c.eps;
  P.at = (float)(1.0 - (double)c.lr * (double)c.weight_decay);
  P.ns = (float)std::sqrt(2.0 * (double)c.lr * (double)c.temperature);
  P.S_total_u = (unsigned long long)h->s.S_total;
  R.c[0] = h->c[0]; R.c[1] = h->c[1];
  R.sums[0] = h->sums[0]; R.sums[1] = h->sums[1]; R.sums[2] = h->sums[2];
  R.p[0] = h->p[0]; R.p[1] = h->p[1];
  R.nbase = mix64_host(c.seed ^ 0x6A09E667F3BCC909ull);
  P.off = c.replica_offset;
  R.S_total = (double)h->s.S_total;
  R.sched = h->sched;
  std::vector<float4> tab((size_t)std::min<int64_t>(n_steps, kSchedCap));
  for (int64_t k0 = 0; k0 < n_steps; k0 += kSchedCap) {
    const int nk = (int)std::min<int64_t>(kSchedCap, n_steps - k0);
    for (int j = 0; j < nk; ++j) {   // the same host double -> fp32 scalars as the launch-per-step path
      const int64_t t = h->step + j + 1;
      tab[j] = make_float4((float)(-2.0 * (double)c.alpha * (double)gamma[k0 + j]),
                           (float)((double)c.lr / (1.0 - std::pow((double)c.beta1, (double)t))),
                           (float)(1.0 / std::sqrt(1.0 - std::pow((double)c.beta2, (double)t))), 0.0f);
    }
    // stream-ordered after the previous chunk's launch (pageable source: staged before return)
    QQA_CUDA(cudaMemcpyAsync(h->sched, tab.data(), (size_t)nk * sizeof(float4), cudaMemcpyHostToDevice, h->stream));
    R.t0 = h->step;
    R.nsteps = nk;
    R.cur0 = h->cur;
    R.scur0 = h->scur;
    void* args[] = {(void*)&R};
    int st;
    if ((st = record_start(h))) return st;
    const cudaError_t le = cudaLaunchCooperativeKernel((const void*)kr, dim3(h->grid_run), dim3(h->run_cta), args,
                                                       0, h->stream);
    if (le == cudaErrorCooperativeLaunchTooLarge) {
      // the grid cannot be co-resident now (e.g. a shared GPU): the launch-per-step path
      // runs the remaining steps (bit-identical) and the handle stops using k_run
      (void)cudaGetLastError();   // (the unmatched start event is re-recorded by the next step)
      h->grid_run = 0;
      return do_steps(h, gamma + k0, n_steps - k0);
    }
    QQA_CUDA(le);
    h->launches++;
    if (h->profiling) {   // one launch = nk steps: per-step kernel time = span / nk
      QQA_CUDA(cudaEventRecord(h->ev[h->ev_used + 1], h->stream));
      h->ev_used += 2;
      h->prof_launches += nk;
    }
    h->cur = (h->cur + nk) & 1;
    h->scur = (int)((h->scur + nk) % 3);
    h->step += nk;
  }
  return QQA_OK;
}

// One-cluster path (k_run_cluster): one GPU, unblocked, n S_p <= kClusterMaxElems. QQA_CLUSTER=0/1
// overrides; an explicit QQA_PERSISTENT selects k_run / k_step instead.
bool use_cluster(const qqa_handle* h, int64_t n_steps) {
  if (h->cluster_cs <= 0 || h->comm || h->xmode || n_steps < 2) return false;
  if (const char* env = std::getenv("QQA_CLUSTER")) return std::atoi(env) != 0;
  return std::getenv("QQA_PERSISTENT") == nullptr;
}

int do_steps_cluster(qqa_handle* h, const float* gamma, int64_t n_steps) {
  const qqa_config& c = h->cfg;
  qqa::RunParams R{};
  qqa::StepParams& P = R.P;
  P.rowptr = h->rowptr; P.rowptr_pad = h->rowptr_pad; P.colidx_pad = h->colidx_pad;
  P.theta = h->theta; P.m = h->m; P.v = h->v; P.flag = h->flag;
  P.n = h->s.n; P.SB = h->s.SB; P.B = h->s.B; P.S_local = h->s.S_local; P.S_total = (double)h->s.S_total;
  P.row_begin = 0; P.row_end = h->s.n;
  P.problem = problem_kind(c.problem);
  P.alpha = c.alpha; P.lam = c.penalty; P.comm = c.comm;
  P.b1 = c.beta1; P.c1 = (float)(1.0 - (double)c.beta1);
  P.b2 = c.beta2; P.c2 = (float)(1.0 - (double)c.beta2);
  P.eps = c.eps;
  P.at = (float)(1.0 - (double)c.lr * (double)c.weight_decay);
  P.ns = (float)std::sqrt(2.0 * (double)c.lr * (double)c.temperature);
  P.S_total_u = (unsigned long long)h->s.S_total;
  P.off = c.replica_offset;
  R.c[0] = h->c[0]; R.c[1] = h->c[1];
  R.sums[0] = h->sums[0]; R.sums[1] = h->sums[1]; R.sums[2] = h->sums[2];
  R.p[0] = h->p[0]; R.p[1] = h->p[1];
  R.nbase = mix64_host(c.seed ^ 0x6A09E667F3BCC909ull);
  R.S_total = (double)h->s.S_total;
  R.sched = h->sched;
  R.rows_cta = h->cluster_rows;
  const qqa::RunKernel kc = qqa::cluster_kernel(step_mode(c, h->s.weighted));
  std::vector<float4> tab((size_t)std::min<int64_t>(n_steps, kSchedCap));
  for (int64_t k0 = 0; k0 < n_steps; k0 += kSchedCap) {
    const int nk = (int)std::min<int64_t>(kSchedCap, n_steps - k0);
    for (int j = 0; j < nk; ++j) {   // the same host double -> fp32 scalars as the other paths
      const int64_t t = h->step + j + 1;
      tab[j] = make_float4((float)(-2.0 * (double)c.alpha * (double)gamma[k0 + j]),
                           (float)((double)c.lr / (1.0 - std::pow((double)c.beta1, (double)t))),
                           (float)(1.0 / std::sqrt(1.0 - std::pow((double)c.beta2, (double)t))), 0.0f);
    }
    QQA_CUDA(cudaMemcpyAsync(h->sched, tab.data(), (size_t)nk * sizeof(float4), cudaMemcpyHostToDevice, h->stream));
    R.t0 = h->step;
    R.nsteps = nk;
    R.cur0 = h->cur;
    R.scur0 = h->scur;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(h->cluster_cs);
    lc.blockDim = dim3(QQA_CLUSTER_CT);
    lc.dynamicSmemBytes = h->cluster_smem;
    lc.stream = h->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = h->cluster_cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int st;
    if ((st = record_start(h))) return st;
    const cudaError_t le = cudaLaunchKernelEx(&lc, kc, R);
    if (le == cudaErrorLaunchOutOfResources || le == cudaErrorCooperativeLaunchTooLarge ||
        le == cudaErrorInvalidClusterSize) {
      // the cluster cannot be placed now (e.g. a shared GPU): the remaining steps run on the other
      // (bit-identical) paths and the handle stops using k_run_cluster
      (void)cudaGetLastError();
      h->cluster_cs = 0;
      return do_steps(h, gamma + k0, n_steps - k0);
    }
    QQA_CUDA(le);
    h->launches++;
    if (h->profiling) {   // one launch = nk steps
      QQA_CUDA(cudaEventRecord(h->ev[h->ev_used + 1], h->stream));
      h->ev_used += 2;
      h->prof_launches += nk;
    }
    h->cur = (h->cur + nk) & 1;
    h->scur = (int)((h->scur + nk) % 3);
    h->step += nk;
  }
  return QQA_OK;
}

// Step-invariant parameters of the fused-exchange step (k_step_x and its one-GPU emulation).
qqa::StepParams xstep_base(const qqa_handle* h) {
  const qqa_config& c = h->cfg;
  qqa::StepParams P{};
  P.rowptr = h->rowptr; P.rowptr_pad = h->rowptr_pad; P.colidx_pad = h->colidx_pad;
  P.w_pad = h->w_pad; P.wdeg = h->wdeg;
  P.theta = h->theta; P.m = h->m; P.v = h->v; P.flag = h->flag;
  P.n = h->s.n; P.SB = h->s.SB; P.B = h->s.B; P.S_local = h->s.S_local; P.S_total = (double)h->s.S_total;
  P.off = c.replica_offset;
  P.row_begin = 0; P.row_end = h->s.n;
  P.problem = problem_kind(c.problem);
  P.alpha = c.alpha; P.lam = c.penalty; P.comm = c.comm;
  P.b1 = c.beta1; P.c1 = (float)(1.0 - (double)c.beta1);
  P.b2 = c.beta2; P.c2 = (float)(1.0 - (double)c.beta2);
  P.eps = c.eps;
  P.at = (float)(1.0 - (double)c.lr * (double)c.weight_decay);
  P.ns = (float)std::sqrt(2.0 * (double)c.lr * (double)c.temperature);
  P.S_total_u = (unsigned long long)h->s.S_total;
  return P;
}

// The per-step part of the fused-exchange step t = h->step + 1 (buffers a -> b, scalars of gamma).
qqa::StepVar xstep_var(const qqa_handle* h, float gamma) {
  const qqa_config& c = h->cfg;
  const int64_t t = h->step + 1;
  qqa::StepVar V{};
  V.nkey = mix64_host(c.seed ^ 0x6A09E667F3BCC909ull) + (uint64_t)t * (uint64_t)h->s.n * (uint64_t)h->s.S_total;
  V.kt = (float)(-2.0 * (double)c.alpha * (double)gamma);
  V.st = (float)((double)c.lr / (1.0 - std::pow((double)c.beta1, (double)t)));
  V.rt = (float)(1.0 / std::sqrt(1.0 - std::pow((double)c.beta2, (double)t)));
  V.p_cur = h->p[h->cur];
  V.p_next = h->p[h->cur ^ 1];
  V.rev = (h->serpentine && h->s.B > 1 && (t & 1)) ? 1 : 0;
  return V;
}

// Fused-exchange steps: one k_step_x launch per step (it waits for the previous step's barrier,
// finalizes from the owners' sums, adds into the owners' next sums and arrives); no NCCL, no k_finalize.
int do_steps_x(qqa_handle* h, const float* gamma, int64_t n_steps) {
  const qqa_config& c = h->cfg;
  const qqa::XStepKernel kx = pick_xstep(h->s.lanes, h->s.vpl, step_mode(c, h->s.weighted), full_lanes(h->s));
  if (!kx) return fail(QQA_ERR_UNSUPPORTED, "no fused-exchange kernel for this mode");
  qqa::StepParams P = xstep_base(h);
  for (int64_t k = 0; k < n_steps; ++k) {
    const int64_t t = h->step + 1;
    P.var = xstep_var(h, gamma[k]);
    const int a = h->cur, b = h->cur ^ 1;
    const int sa = h->scur, sb = (h->scur + 1) % 3, sz = (h->scur + 2) % 3;
    if (h->s.n > 0) {
      const qqa::XParams X = make_xparams(h, sa, sb, sz, a, b);
      int st;
      if ((st = record_start(h))) return st;
      kx<<<h->grid_step, 256, 0, h->stream>>>(P, X);
      QQA_CUDA(cudaGetLastError());
      h->launches++;
      h->xsync++;
      if ((st = record_end(h))) return st;
    }
    h->cur = b;
    h->scur = sb;
    h->step = t;
  }
  return QQA_OK;
}

// Owner-slotted exchange steps: one cooperative k_step_xs launch per step (two barrier arrivals each:
// after the owner reduction and after the step).
int do_steps_xs(qqa_handle* h, const float* gamma, int64_t n_steps) {
  const qqa::XStepKernel kx = pick_xsstep(h->s.lanes, h->s.vpl, step_mode(h->cfg, h->s.weighted), full_lanes(h->s));
  if (!kx || h->grid_xs <= 0) return fail(QQA_ERR_UNSUPPORTED, "no owner-slotted exchange kernel for this layout");
  qqa::StepParams P = xstep_base(h);
  for (int64_t k = 0; k < n_steps; ++k) {
    const int64_t t = h->step + 1;
    P.var = xstep_var(h, gamma[k]);
    const int a = h->cur, b = h->cur ^ 1;
    const int sb = (h->scur + 1) % 3;
    if (h->s.n > 0) {
      qqa::XParams X = make_xparams(h, h->scur, sb, (h->scur + 2) % 3, a, b);
      void* args[] = {(void*)&P, (void*)&X};
      int st;
      if ((st = record_start(h))) return st;
      QQA_CUDA(cudaLaunchCooperativeKernel((const void*)kx, dim3(h->grid_xs), dim3(256), args, 0, h->stream));
      h->launches++;
      h->xsync += 2;
      if ((st = record_end(h))) return st;
    }
    h->cur = b;
    h->scur = sb;
    h->step = t;
  }
  return QQA_OK;
}

int do_steps(qqa_handle* h, const float* gamma, int64_t n_steps) {
  if (n_steps < 0) return fail(QQA_ERR_INVALID_ARG, "n_steps < 0");
  if (n_steps > 0 && !gamma) return fail(QQA_ERR_INVALID_ARG, "gamma is NULL");
  if (h->s.kary) return do_steps_kary(h, gamma, n_steps);
  if (h->xmode) return h->xslotted ? do_steps_xs(h, gamma, n_steps) : do_steps_x(h, gamma, n_steps);
  if (use_cluster(h, n_steps)) return do_steps_cluster(h, gamma, n_steps);
  if (use_persistent(h, n_steps)) return do_steps_persistent(h, gamma, n_steps);
  StepKernel ks;
  InitKernel ki;
  pick_kernels(h->s.lanes, h->s.vpl, step_mode(h->cfg, h->s.weighted), ks, ki, nullptr, 256, full_lanes(h->s));
  const qqa_config& c = h->cfg;
  qqa::StepParams P{};
  P.rowptr = h->rowptr; P.rowptr_pad = h->rowptr_pad; P.colidx_pad = h->colidx_pad;
  P.w_pad = h->w_pad; P.wdeg = h->wdeg;
  P.theta = h->theta; P.m = h->m; P.v = h->v; P.flag = h->flag;
  P.n = h->s.n; P.SB = h->s.SB; P.B = h->s.B; P.S_local = h->s.S_local; P.S_total = (double)h->s.S_total;
  P.off = c.replica_offset;
  P.problem = problem_kind(c.problem);  // dense clique = MIS on the complement
  P.alpha = c.alpha; P.lam = c.penalty; P.comm = c.comm;
  P.b1 = c.beta1; P.c1 = (float)(1.0 - (double)c.beta1);
  P.b2 = c.beta2; P.c2 = (float)(1.0 - (double)c.beta2);
  P.eps = c.eps;
  P.ns = (float)std::sqrt(2.0 * (double)c.lr * (double)c.temperature);   // Eq. 9: sqrt(2 eta T)
  P.S_total_u = (unsigned long long)h->s.S_total;
  P.blo = 0; P.bhi = h->s.B;
  const uint64_t nbase = mix64_host(c.seed ^ 0x6A09E667F3BCC909ull);    // noise stream
  for (int64_t k = 0; k < n_steps; ++k) {
    const int64_t t = h->step + 1;  // Adam step index (reading R11)
    // xi key of (t, i, global s) = nbase + (t n + i) S_total + s_even  (mod 2^64; replica pairs, R24)
    P.var.nkey = nbase + (uint64_t)t * (uint64_t)h->s.n * (uint64_t)h->s.S_total;
    P.var.kt = (float)(-2.0 * (double)c.alpha * (double)gamma[k]);
    P.at = (float)(1.0 - (double)c.lr * (double)c.weight_decay);
    P.var.st = (float)((double)c.lr / (1.0 - std::pow((double)c.beta1, (double)t)));
    P.var.rt = (float)(1.0 / std::sqrt(1.0 - std::pow((double)c.beta2, (double)t)));
    const int a = h->cur, b = h->cur ^ 1;
    const int sa = h->scur, sb = (h->scur + 1) % 3, sz = (h->scur + 2) % 3;
    P.var.p_cur = h->p[a]; P.var.p_next = h->p[b];
    P.var.rev = (h->serpentine && h->s.B > 1 && (t & 1)) ? 1 : 0;
    P.ms = h->ms;
    P.colsum = h->colsum[a];
    P.var.sums_next = h->sums[sb];
    P.var.sums_zero = (h->s.B > 1) ? h->sums[sz] : nullptr;
    const int C = (h->comm && h->s.n > 0) ? h->comm_chunks : 1;
    if (h->s.n > 0) {
      // K0: (mu_i, STD_i) of the current p, shift of the next sums
      qqa::k_finalize<<<h->grid_fin, 256, 0, h->stream>>>(h->c[a], h->sums[sa], h->s.n, (double)h->s.S_total,
                                                           h->ms, h->c[b]);
      QQA_CUDA(cudaGetLastError());
      h->launches++;
      int st;
      if ((st = record_start(h))) return st;
      if (h->s.KS > 1) {   // segmented gather: per replica block, KS - 1 partial passes, then the last + update
        const int KS = h->s.KS;
        for (int bq = 0; bq < h->s.B; ++bq) {
          qqa::StepParams Q = P;
          Q.blo = bq; Q.bhi = bq + 1;
          Q.colidx_pad = h->colidx_seg;
          for (int k = 0; k < KS; ++k) {
            Q.rowptr_pad = h->rowptr_seg + (size_t)k * ((size_t)h->s.n + 1);
            const int q = (k == 0) ? 0 : (k < KS - 1) ? 1 : 2;
            if (k == KS - 1 && C > 1) break;   // chunked last pass below (communicator overlap)
            Q.row_begin = 0; Q.row_end = h->s.n;
            h->kseg[q]<<<h->grid_seg[q], 256, 0, h->stream>>>(Q);
            QQA_CUDA(cudaGetLastError());
            h->launches++;
          }
        }
      }
      for (int ch = 0; ch < C; ++ch) {
        P.row_begin = (int)((int64_t)h->s.n * ch / C);
        P.row_end = (int)((int64_t)h->s.n * (ch + 1) / C);
        if (h->s.KS > 1) {
          if (C == 1) break;   // every pass already launched above
          qqa::StepParams Q = P;
          Q.blo = 0; Q.bhi = h->s.B;
          Q.colidx_pad = h->colidx_seg;
          Q.rowptr_pad = h->rowptr_seg + (size_t)(h->s.KS - 1) * ((size_t)h->s.n + 1);
          h->kseg[2]<<<h->grid_seg[2], 256, 0, h->stream>>>(Q);
        } else if (h->kst)
          h->kst<<<h->grid_st, 256, h->st_smem, h->stream>>>(P);
        else
          ks<<<h->grid_step, 256, 0, h->stream>>>(P);
        QQA_CUDA(cudaGetLastError());
        h->launches++;
        if (C > 1) {  // all-reduce this chunk's rows on the comm stream while the next chunk computes
          QQA_CUDA(cudaEventRecord(h->chunk_ev[ch], h->stream));
          QQA_CUDA(cudaStreamWaitEvent(h->cstream, h->chunk_ev[ch], 0));
          const size_t r0 = (size_t)P.row_begin, rows = (size_t)(P.row_end - P.row_begin);
          QQA_NCCL(ncclGroupStart());
          QQA_NCCL(ncclAllReduce(h->sums[sb] + r0, h->sums[sb] + r0, rows, ncclInt64, ncclSum, h->comm, h->cstream));
          QQA_NCCL(ncclAllReduce(h->sums[sb] + h->s.n + r0, h->sums[sb] + h->s.n + r0, rows, ncclInt64, ncclSum,
                                 h->comm, h->cstream));
          QQA_NCCL(ncclGroupEnd());
        }
      }
      if ((st = record_end(h))) return st;
      if (c.problem == QQA_MAXCLIQUE_SPARSE && (st = launch_colsum(h, b))) return st;
      if (C > 1) {  // the next step's finalize needs every chunk's reduced sums
        QQA_CUDA(cudaEventRecord(h->chunk_ev[C], h->cstream));
        QQA_CUDA(cudaStreamWaitEvent(h->stream, h->chunk_ev[C], 0));
      }
    }
    if (h->comm && C == 1) {
      QQA_NCCL(ncclAllReduce(h->sums[sb], h->sums[sb], 2 * (size_t)h->s.n, ncclInt64, ncclSum, h->comm, h->stream));
    }
    h->cur = b;
    h->scur = sb;
    h->step = t;
  }
  return QQA_OK;
}

// Host [n][S_local] <-> device [B][n][SB], one 2-D copy per replica block.
// K-ary: host [n][S_local][K] <-> device [n][S_local][KP], one 2-D copy.
int copy_blocked(qqa_handle* h, float* host, float* dev, cudaMemcpyKind dir) {
  const Shape& s = h->s;
  if (s.n == 0) return QQA_OK;
  if (s.kary) {
    const size_t rows = (size_t)s.n * s.S_local, hp = (size_t)s.K * sizeof(float), dp = (size_t)s.KP * sizeof(float);
    if (dir == cudaMemcpyDeviceToHost)
      QQA_CUDA(cudaMemcpy2DAsync(host, hp, dev, dp, hp, rows, dir, h->stream));
    else
      QQA_CUDA(cudaMemcpy2DAsync(dev, dp, host, hp, hp, rows, dir, h->stream));
    return QQA_OK;
  }
  for (int b = 0; b < s.B; ++b) {
    const int cols = std::min(s.SB, s.S_local - b * s.SB);
    if (cols <= 0) break;
    float* hb = host + (size_t)b * s.SB;
    float* db = dev + (size_t)b * ((size_t)s.n + 1) * s.SB;
    if (dir == cudaMemcpyDeviceToHost)
      QQA_CUDA(cudaMemcpy2DAsync(hb, (size_t)s.S_local * sizeof(float), db, (size_t)s.SB * sizeof(float),
                                 (size_t)cols * sizeof(float), (size_t)s.n, dir, h->stream));
    else
      QQA_CUDA(cudaMemcpy2DAsync(db, (size_t)s.SB * sizeof(float), hb, (size_t)s.S_local * sizeof(float),
                                 (size_t)cols * sizeof(float), (size_t)s.n, dir, h->stream));
  }
  return QQA_OK;
}

int set_device(qqa_handle* h) {
  int cur = -1;
  QQA_CUDA(cudaGetDevice(&cur));
  if (cur != h->device) QQA_CUDA(cudaSetDevice(h->device));
  return QQA_OK;
}

// Chunked compute / all-reduce overlap for the binary step (K-ary keeps one all-reduce per
// step). QQA_COMM_CHUNKS overrides the default: 2 chunks with > 1 rank, none with one. Measured on
// c5's G = 8 shard (S_l = 8, one rank, profiles/r2_host_enqueue.txt): every extra chunk launch costs
// device time (131 / 144 / 162 / 177 us per step for 1 / 2 / 3 / 4 chunks), more than the ~1/C of a
// 16 MB all-reduce (~40-55 us at G = 8) each further chunk would hide, so 2.
int setup_overlap(qqa_handle* h) {
  int C = (h->nranks > 1 && !h->s.kary) ? 2 : 1;
  if (const char* env = std::getenv("QQA_COMM_CHUNKS")) C = std::max(1, std::min(64, std::atoi(env)));
  if (h->s.kary || h->s.n < C) C = 1;
  h->comm_chunks = C;
  if (C > 1 && !h->cstream) {
    int lo = 0, hi = 0;
    QQA_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    QQA_CUDA(cudaStreamCreateWithPriority(&h->cstream, cudaStreamNonBlocking, hi));   // comm first
  }
  while ((int)h->chunk_ev.size() < C + 1) {
    cudaEvent_t e;
    QQA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->chunk_ev.push_back(e);
  }
  return QQA_OK;
}

}  // namespace

extern "C" {

int qqa_version(void) { return QQA_ABI_VERSION; }

const char* qqa_last_error(void) { return g_last_error.c_str(); }

const char* qqa_status_string(int status) {
  switch (status) {
    case QQA_OK: return "ok";
    case QQA_ERR_INVALID_ARG: return "invalid argument";
    case QQA_ERR_BAD_GRAPH: return "bad graph";
    case QQA_ERR_CUDA: return "cuda error";
    case QQA_ERR_COMM: return "communication error";
    case QQA_ERR_NONFINITE: return "non-finite value";
    case QQA_ERR_UNSUPPORTED: return "unsupported";
    case QQA_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int qqa_workspace_bytes(const qqa_graph* g, const qqa_config* cfg, size_t* bytes) {
  if (!bytes) return fail(QQA_ERR_INVALID_ARG, "bytes is NULL");
  Shape s;
  int st = make_shape(g, cfg, s);
  if (st) return st;
  *bytes = make_layout(s).total;
  return QQA_OK;
}

int qqa_create(qqa_handle** out, const qqa_graph* g, const qqa_config* cfg, void* d_workspace,
               size_t workspace_bytes, void* stream) {
  NvtxRange nvtx("qqa_create");
  if (!out) return fail(QQA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  Shape s;
  int st = make_shape(g, cfg, s);
  if (st) return st;
  const Layout L = make_layout(s);
  if (!d_workspace || ((uintptr_t)d_workspace % kAlign) != 0)
    return fail(QQA_ERR_WORKSPACE, "workspace is NULL or not 256-byte aligned");
  if (workspace_bytes < L.total)
    return fail(QQA_ERR_WORKSPACE, "workspace has " + std::to_string(workspace_bytes) + " bytes, needs " +
                                       std::to_string(L.total));
  int dev = 0, ndev = 0;
  QQA_CUDA(cudaGetDeviceCount(&ndev));
  QQA_CUDA(cudaGetDevice(&dev));
  cudaPointerAttributes attr{};
  QQA_CUDA(cudaPointerGetAttributes(&attr, d_workspace));
  if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
    return fail(QQA_ERR_WORKSPACE, "workspace is not device memory");

  qqa_handle* h = new qqa_handle();
  h->device = attr.device;
  h->stream = (cudaStream_t)stream;
  h->cfg = *cfg;
  h->s = s;
  h->L = L;
  auto cleanup = [&](int status) { delete h; return status; };
  if ((st = set_device(h))) return cleanup(st);
  {
    cudaError_t e = cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device);
    if (e != cudaSuccess) return cleanup(fail(QQA_ERR_CUDA, cudaGetErrorString(e)));
  }
  char* ws = (char*)d_workspace;
  h->ws = ws;
  h->rowptr = (int*)(ws + L.rowptr);
  h->colidx = (int*)(ws + L.colidx);
  h->rowptr_pad = (int*)(ws + L.rowptr_pad);
  h->colidx_pad = (int*)(ws + L.colidx_pad);
  h->theta = (float*)(ws + L.theta);
  h->m = (float*)(ws + L.m);
  h->v = (float*)(ws + L.v);
  h->p[0] = (float*)(ws + L.p0);
  h->p[1] = (float*)(ws + L.p1);
  h->c[0] = (float*)(ws + L.c0);
  h->c[1] = (float*)(ws + L.c1);
  h->sums[0] = (long long*)(ws + L.s0);
  h->sums[1] = (long long*)(ws + L.s1);
  h->sums[2] = (long long*)(ws + L.s2);
  h->ms = (float2*)(ws + L.ms);
  h->flag = (int*)(ws + L.flag);
  h->X = (uint32_t*)(ws + L.X);
  h->counts = (unsigned long long*)(ws + L.counts);
  h->tot = (long long*)(ws + L.tot);
  h->energy = (double*)(ws + L.energy);
  h->best = (int*)(ws + L.best);
  h->beste = (double*)(ws + L.beste);
  h->genergy = (double*)(ws + L.genergy);
  h->gbest = (int*)(ws + L.gbest);
  h->gbeste = (double*)(ws + L.gbeste);
  h->gor = g->group_of_row ? (int*)(ws + L.gor) : nullptr;
  h->xbuf = (uint8_t*)(ws + L.xbuf);
  h->sched = (float4*)(ws + L.sched);
  h->colsum[0] = (long long*)(ws + L.cs0);
  h->colsum[1] = (long long*)(ws + L.cs1);
  if (s.weighted) {
    h->w = (float*)(ws + L.w);
    h->w_pad = (float*)(ws + L.w_pad);
    h->wdeg = (float*)(ws + L.wdeg);
  }
  h->wsums = (long long*)(ws + L.wsums);
  if (const char* env = std::getenv("QQA_SERPENTINE")) h->serpentine = std::atoi(env) != 0;

  // Graph -> device (int32 offsets). Max clique walks the complement graph.
  std::vector<int> rp32, ci_c;
  const int32_t* ci_src = g->colidx;
  if (cfg->problem == QQA_MAXCLIQUE) {
    if ((st = validate_host(g))) return cleanup(st);
    build_complement(g, rp32, ci_c);
    if ((int64_t)ci_c.size() != s.nnz || rp32[s.n] != (int)s.nnz)   // the sizes make_shape planned
      return cleanup(fail(QQA_ERR_BAD_GRAPH, "graph rejected: complement size differs from the planned one"));
    ci_src = ci_c.data();
  } else {
    rp32.resize((size_t)s.n + 1);
    for (int i = 0; i <= s.n; ++i) rp32[i] = (int)(s.n ? g->rowptr[i] : 0);
  }
#define QQA_CUDA_C(call)                                                                        \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return cleanup(fail(QQA_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)));   \
  } while (0)
  QQA_CUDA_C(cudaMemcpyAsync(h->rowptr, rp32.data(), rp32.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  if (s.nnz > 0)
    QQA_CUDA_C(cudaMemcpyAsync(h->colidx, ci_src, (size_t)s.nnz * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  if (h->gor && s.n > 0)
    QQA_CUDA_C(cudaMemcpyAsync(h->gor, g->group_of_row, (size_t)s.n * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  if (h->w && s.nnz > 0)
    QQA_CUDA_C(cudaMemcpyAsync(h->w, g->weights, (size_t)s.nnz * sizeof(float), cudaMemcpyHostToDevice, h->stream));
  QQA_CUDA_C(cudaMemsetAsync(h->flag, 0, 4 * sizeof(int), h->stream));
  // theta/m/v padding and the zero row n of both p buffers (K-ary: the colour padding)
  if (s.kary) {
    h->theta = nullptr;
    for (float* buf : {h->m, h->v, h->p[0], h->p[1]})
      QQA_CUDA_C(cudaMemsetAsync(buf, 0, (size_t)s.n * s.S_local * s.KP * sizeof(float), h->stream));
  } else {
    for (float* buf : {h->theta, h->m, h->v, h->p[0], h->p[1]})
      QQA_CUDA_C(cudaMemsetAsync(buf, 0, ((size_t)s.n + 1) * s.S_p * sizeof(float), h->stream));
  }
  if (cfg->problem != QQA_MAXCLIQUE && s.n > 0 && s.nnz > 0) {
    const int blocks = std::max(1, std::min((s.n + 255) / 256, h->sm_count * 8));
    qqa::k_validate<<<blocks, 256, 0, h->stream>>>(h->rowptr, h->colidx, s.n, h->gor, h->w, h->flag);
    QQA_CUDA_C(cudaGetLastError());
    h->launches++;
    int flag = 0;
    QQA_CUDA_C(cudaMemcpyAsync(&flag, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    QQA_CUDA_C(cudaStreamSynchronize(h->stream));
    if (flag) {
      std::string why;
      if (flag & 2) why += " column out of range;";
      if (flag & 4) why += " row not strictly ascending (unsorted or duplicate);";
      if (flag & 8) why += " self-loop;";
      if (flag & 16) why += " not symmetric;";
      if (flag & 32) why += " edge between two instances of the batch;";
      if (flag & 64) why += " asymmetric (w_ij != w_ji) or non-finite edge weight;";
      return cleanup(fail(QQA_ERR_BAD_GRAPH, "graph rejected:" + why));
    }
  }
  {  // row-padded CSR for the step kernel (rows rounded up to 4 entries, sentinel n)
    std::vector<int> rp_pad((size_t)s.n + 1, 0);
    for (int i = 0; i < s.n; ++i) rp_pad[i + 1] = rp_pad[i] + (rp32[i + 1] - rp32[i] + 3) / 4 * 4;
    if ((int64_t)rp_pad[s.n] != s.nnz_pad)
      return cleanup(fail(QQA_ERR_BAD_GRAPH, "graph rejected: padded CSR size differs from the planned one"));
    QQA_CUDA_C(cudaMemcpyAsync(h->rowptr_pad, rp_pad.data(), rp_pad.size() * sizeof(int), cudaMemcpyHostToDevice,
                               h->stream));
    if (s.n > 0) {
      const int blocks = std::max(1, std::min((s.n + 255) / 256, h->sm_count * 8));
      qqa::k_pad_csr<<<blocks, 256, 0, h->stream>>>(h->rowptr, h->colidx, h->rowptr_pad, h->colidx_pad, s.n, h->w,
                                                    h->w_pad, h->wdeg);
      QQA_CUDA_C(cudaGetLastError());
      h->launches++;
    }
    QQA_CUDA_C(cudaStreamSynchronize(h->stream));  // rp_pad is pageable host memory
  }
  if (s.KS > 1) {  // segmented gather: segment CSRs (built on the host from the validated graph) and kernels
    std::vector<int> rps((size_t)s.KS * ((size_t)s.n + 1)), cis((size_t)s.nnz_seg);
    if (build_seg_csr(g->rowptr, g->colidx, s.n, s.KS, rps.data(), cis.data()) != s.nnz_seg)
      return cleanup(fail(QQA_ERR_BAD_GRAPH, "graph rejected: segment CSR size differs from the planned one"));
    h->rowptr_seg = (int*)(ws + L.rowptr_seg);
    h->colidx_seg = (int*)(ws + L.colidx_seg);
    QQA_CUDA_C(cudaMemcpyAsync(h->rowptr_seg, rps.data(), rps.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    QQA_CUDA_C(cudaMemcpyAsync(h->colidx_seg, cis.data(), cis.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    if (!qqa::seg_kernels(s.lanes, step_mode(*cfg, s.weighted), h->kseg[0], h->kseg[1], h->kseg[2]))
      return cleanup(fail(QQA_ERR_UNSUPPORTED, "no segmented-gather kernel for this shape"));
    for (int q = 0; q < 3; ++q)
      if ((st = grid_for((const void*)h->kseg[q], h->sm_count, s.n, s.lanes, h->grid_seg[q]))) return cleanup(st);
    QQA_CUDA_C(cudaStreamSynchronize(h->stream));   // rps / cis are pageable host memory
  }
  if (s.kary) {
    StepKKernel ks;
    InitKKernel ki;
    PackKKernel kp;
    if (!pick_kary(s.KP, s.K, step_mode(*cfg, s.weighted), ks, ki, kp)) return cleanup(fail(QQA_ERR_UNSUPPORTED, "no K-ary kernel"));
    const int64_t chunks = (s.S_local + s.LK - 1) / s.LK;   // work item = (variable, replica chunk)
    if ((st = grid_for((const void*)ks, h->sm_count, (int64_t)s.n * chunks, s.LK, h->grid_step))) return cleanup(st);
    {  // colour quads for KP 12 / 16 (QQA_KARY_QUAD=0 keeps k_step_K)
      const char* env = std::getenv("QQA_KARY_QUAD");
      // KP = 8 (2 lanes per replica) only with QQA_KARY_QUAD=2 (experiment)
      const int qsel = env ? std::atoi(env) : 1;
      h->kq = (qsel == 0 || (s.KP == 8 && qsel != 2)) ? nullptr : qqa::kary_quad_kernel(s.KP, step_mode(*cfg, s.weighted));
      if (h->kq) {
        const int reps = qqa::kary_quad_reps(s.KP);   // replicas per warp (16 for KP = 8: two items)
        const int64_t qitems = ((int64_t)s.n * ((s.S_local + qqa::kQuadReps - 1) / qqa::kQuadReps) * qqa::kQuadReps + reps - 1) / reps;
        if ((st = grid_for((const void*)h->kq, h->sm_count, qitems, 32, h->grid_kq))) return cleanup(st);
      }
    }
    if ((st = grid_for((const void*)ki, h->sm_count, (int64_t)s.n * s.S_local, 1, h->grid_init))) return cleanup(st);
    const int64_t nk = (int64_t)s.n * s.K;
    h->grid_fin = (int)std::max<int64_t>(1, std::min<int64_t>((nk + 255) / 256, (int64_t)h->sm_count * 8));
  } else {
    StepKernel ks;
    InitKernel ki;
    RunKernel kr = nullptr;
    // contiguous-row persistent CTAs when the kernel fits 64 registers (VPL 1) and the work
    // fills every SM with a 1024-thread CTA (measured: profiles/r1_design_iterations.md)
    // contiguous rows per SM pay off for a batch of small instances (an SM's rows are about one instance,
    // whose p rows stay in L1: c2 53.0 vs 56.7 us with 256-thread CTAs), best as one 768-thread CTA per SM with
    // up to 85 registers (c2 48.8 vs 53.2 at 1024 threads and 64 registers; t1 353.0 vs 351.5); a single random
    // graph has no such locality and runs 3 x 256 threads per SM (c3 19.9 vs 20.9 at 768, 22.8 at 1024;
    // profiles/r2_ab_run256_minb.txt, r2_ab_run768.txt)
    h->run_cta = (s.vpl == 1 && s.G > 1 && (int64_t)s.n * s.lanes >= (int64_t)h->sm_count * 768) ? 768 : 256;
    if (const char* env = std::getenv("QQA_RUN_CTA")) {
      const int c = std::atoi(env);
      h->run_cta = (s.vpl == 1 && (c == 1024 || c == 768)) ? c : 256;
    }
    if (!pick_kernels(s.lanes, s.vpl, step_mode(*cfg, s.weighted), ks, ki, &kr, h->run_cta, full_lanes(s)))
      return cleanup(fail(QQA_ERR_UNSUPPORTED, "no kernel for this S_local"));
    if ((st = grid_for((const void*)ks, h->sm_count, s.n, s.lanes, h->grid_step))) return cleanup(st);
    if (const char* env = std::getenv("QQA_STEP_CARVEOUT")) {   // experiment: L1 / shared split of k_step
      QQA_CUDA_C(cudaFuncSetAttribute((const void*)ks, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(env)));
    }
    {  // persistent kernel: every CTA must be co-resident (cooperative launch)
      int coop = 0;
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device);
      if (coop && s.B == 1 && kr) {   // (no k_run for the printed clique relaxation)
        // no shared memory in k_run: give the SM's unified L1 / shared storage to L1
        QQA_CUDA_C(cudaFuncSetAttribute((const void*)kr, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
        if ((st = grid_for((const void*)kr, h->sm_count, s.n, s.lanes, h->grid_run, h->run_cta)))
          return cleanup(st);
      }
    }
    h->grid_fin = std::max(1, std::min((s.n + 255) / 256, h->sm_count * 8));
    if ((st = grid_for((const void*)ki, h->sm_count, s.n, s.lanes, h->grid_init))) return cleanup(st);
    {  // staged-state step kernel (VPL 1, FULL shapes, modes 0-3), opt-in (QQA_STAGE=1): measured slower on
       // c5 (873 vs 812 us per step; its 32 KB of shared memory per CTA takes L1 space the in-flight gathers
       // use, profiles/r2_design_iterations.md)
      const int mode = step_mode(*cfg, s.weighted);
      bool want = false;
      if (const char* env = std::getenv("QQA_STAGE")) want = std::atoi(env) != 0;
      if (want && s.vpl == 1 && full_lanes(s) && mode <= 3) {
        qqa::StepKernel kt = mode == 0 ? qqa::stage_kernel_m0(s.lanes) : mode == 1 ? qqa::stage_kernel_m1(s.lanes)
                           : mode == 2 ? qqa::stage_kernel_m2(s.lanes) : qqa::stage_kernel_m3(s.lanes);
        if (kt) {
          const size_t smem = 8 * 256 * sizeof(float4);   // [4 vectors][2 halves][256 threads] x 16 B
          int per_sm = 0;
          QQA_CUDA_C(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kt, 256, smem));
          if (per_sm > 0) {
            h->kst = kt;
            h->st_smem = smem;
            const int need = (int)std::max<int64_t>(1, ((int64_t)s.n * s.lanes + 255) / 256);
            h->grid_st = std::max(1, std::min(need, per_sm * h->sm_count));
          }
        }
      }
    }
    if (s.B == 1 && !s.weighted && cfg->problem != QQA_MAXCLIQUE_SPARSE && s.n > 0 &&
        (int64_t)s.n * s.S_p <= kClusterMaxElems && s.nnz_pad * s.S_p <= kClusterMaxGather) {   // tiny: one cluster
      const qqa::RunKernel kc = qqa::cluster_kernel(step_mode(*cfg, s.weighted));
      for (int cs : {16, 8}) {
        if (!kc) break;
        const int rows = next_pow2((s.n + cs - 1) / cs);   // power of two: owner = j >> log2(rows)
        const size_t smem = qqa::cluster_smem_bytes(rows, s.S_p);
        if (smem > 200 * 1024) continue;
        if (cudaFuncSetAttribute((const void*)kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            (cs > 8 && cudaFuncSetAttribute((const void*)kc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                           cudaSuccess)) {
          (void)cudaGetLastError();
          continue;
        }
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(cs);
        lc.blockDim = dim3(QQA_CLUSTER_CT);
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)kc, &lc) != cudaSuccess || nclusters < 1) {
          (void)cudaGetLastError();
          continue;
        }
        h->cluster_cs = cs;
        h->cluster_rows = rows;
        h->cluster_smem = smem;
        break;
      }
    }
  }
  if ((st = launch_init(h, false, nullptr))) return cleanup(st);
  QQA_CUDA_C(cudaStreamSynchronize(h->stream));
#undef QQA_CUDA_C
  *out = h;
  return QQA_OK;
}

int qqa_reset(qqa_handle* h) {
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  h->step = 0;
  return launch_init(h, false, nullptr);
}

int qqa_nccl_unique_id(uint8_t out[128]) {
  if (!out) return fail(QQA_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  QQA_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, 128);
  return QQA_OK;
}

int qqa_attach_comm(qqa_handle* h, const uint8_t id[128], int rank, int nranks) {
  if (!h || !id) return fail(QQA_ERR_INVALID_ARG, "handle or id is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(QQA_ERR_INVALID_ARG, "bad rank / nranks");
  if ((int64_t)h->s.S_local * nranks != h->s.S_total || h->cfg.replica_offset != rank * h->s.S_local)
    return fail(QQA_ERR_INVALID_ARG, "sharding must be S_total = nranks * S_local and replica_offset = rank * S_local");
  int st = set_device(h);
  if (st) return st;
  h->comm_box.reset();
  h->comm = nullptr;
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  QQA_NCCL(ncclCommInitRank(&comm, nranks, uid, rank));
  h->comm_box = std::shared_ptr<ncclComm_t>(new ncclComm_t(comm), [](ncclComm_t* c) {
    ncclCommDestroy(*c);
    delete c;
  });
  h->comm = comm;
  h->rank = rank;
  h->nranks = nranks;
  h->step = 0;
  if ((st = setup_overlap(h))) return st;
  if ((st = launch_init(h, false, nullptr))) return st;
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  return QQA_OK;
}

int qqa_share_comm(qqa_handle* h, qqa_handle* donor) {
  if (!h || !donor) return fail(QQA_ERR_INVALID_ARG, "handle or donor is NULL");
  if (!donor->comm) return fail(QQA_ERR_INVALID_ARG, "donor has no communicator");
  if (donor->device != h->device) return fail(QQA_ERR_INVALID_ARG, "donor lives on another device");
  const int rank = donor->rank, nranks = donor->nranks;
  if ((int64_t)h->s.S_local * nranks != h->s.S_total || h->cfg.replica_offset != rank * h->s.S_local)
    return fail(QQA_ERR_INVALID_ARG, "sharding must be S_total = nranks * S_local and replica_offset = rank * S_local");
  int st = set_device(h);
  if (st) return st;
  h->comm_box = donor->comm_box;
  h->comm = donor->comm;
  h->rank = rank;
  h->nranks = nranks;
  h->step = 0;
  if ((st = setup_overlap(h))) return st;
  if ((st = launch_init(h, false, nullptr))) return st;   // collective: every rank's statistics
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  return QQA_OK;
}

int qqa_run(qqa_handle* h, const float* gamma_host, int64_t n_steps) {
  NvtxRange nvtx("qqa_run");
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  return do_steps(h, gamma_host, n_steps);
}

}  // extern "C"

namespace {

// Loopback exchange: add the current statistic sums of all shards (on one device and stream) and
// write the total back to every shard -- what the NCCL all-reduce does across GPUs.
int loopback_reduce(qqa_handle** hs, int G) {
  qqa_handle* h0 = hs[0];
  const Shape& s = h0->s;
  const long long len = 2 * (long long)s.n * (s.kary ? s.K : 1);
  if (len == 0) return QQA_OK;
  long long* acc = h0->sums[h0->scur];
  const int blocks = (int)std::max<long long>(1, std::min<long long>((len + 255) / 256, (long long)h0->sm_count * 8));
  for (int r = 1; r < G; ++r) {
    qqa::k_add_i64<<<blocks, 256, 0, h0->stream>>>(acc, hs[r]->sums[hs[r]->scur], len);
    QQA_CUDA(cudaGetLastError());
  }
  for (int r = 1; r < G; ++r)
    QQA_CUDA(cudaMemcpyAsync(hs[r]->sums[hs[r]->scur], acc, (size_t)len * sizeof(long long), cudaMemcpyDeviceToDevice,
                             h0->stream));
  return QQA_OK;
}

int check_loopback(qqa_handle** hs, int G) {
  if (!hs || G < 1) return fail(QQA_ERR_INVALID_ARG, "handles is NULL or G < 1");
  for (int r = 0; r < G; ++r) {
    if (!hs[r]) return fail(QQA_ERR_INVALID_ARG, "a handle is NULL");
    const qqa_handle* h = hs[r];
    if (h->comm) return fail(QQA_ERR_INVALID_ARG, "loopback shards must not have a communicator");
    if (h->device != hs[0]->device || h->stream != hs[0]->stream)
      return fail(QQA_ERR_INVALID_ARG, "loopback shards must share one device and one stream");
    if (h->s.n != hs[0]->s.n || h->s.S_local != hs[0]->s.S_local || h->s.S_total != G * h->s.S_local ||
        h->cfg.replica_offset != r * h->s.S_local || h->s.kary != hs[0]->s.kary || h->s.K != hs[0]->s.K ||
        h->scur != hs[0]->scur || h->step != hs[0]->step)
      return fail(QQA_ERR_INVALID_ARG, "loopback shards must be r = 0..G-1 of S_total = G S_local, in lockstep");
  }
  return QQA_OK;
}

}  // namespace

extern "C" {

int qqa_loopback_sync_init(qqa_handle** hs, int G) {
  int st = check_loopback(hs, G);
  if (st) return st;
  if ((st = set_device(hs[0]))) return st;
  if (hs[0]->xslotted) {   // owner-slotted shards: every buffer is zeroed now; scatter the partials, arrive
    for (int r = 0; r < G; ++r) {
      if (!hs[r]->xdefer_init) continue;
      if ((st = xs_scatter_init(hs[r]))) return st;
      if ((st = x_arrive(hs[r]))) return st;
      hs[r]->xdefer_init = false;
    }
    QQA_CUDA(cudaStreamSynchronize(hs[0]->stream));
    return QQA_OK;
  }
  if ((st = loopback_reduce(hs, G))) return st;
  for (int r = 0; r < G; ++r)   // fused-exchange shards: the totals are in place, first barrier
    if (hs[r]->xmode && (st = x_arrive(hs[r]))) return st;
  QQA_CUDA(cudaStreamSynchronize(hs[0]->stream));
  return QQA_OK;
}

int qqa_loopback_run(qqa_handle** hs, int G, const float* gamma_host, int64_t n_steps) {
  NvtxRange nvtx("qqa_loopback_run");
  int st = check_loopback(hs, G);
  if (st) return st;
  if ((st = set_device(hs[0]))) return st;
  if (n_steps > 0 && !gamma_host) return fail(QQA_ERR_INVALID_ARG, "gamma is NULL");
  for (int64_t k = 0; k < n_steps; ++k) {
    for (int r = 0; r < G; ++r)   // one launch-per-step step of every shard (n_steps = 1: no k_run)
      if ((st = do_steps(hs[r], gamma_host + k, 1))) return st;
    if (!hs[0]->xmode && (st = loopback_reduce(hs, G))) return st;   // fused shards exchanged in-kernel
  }
  QQA_CUDA(cudaStreamSynchronize(hs[0]->stream));
  return QQA_OK;
}

int qqa_exchange_emulate(qqa_handle** hs, int G, const float* gamma_host, int64_t n_steps) {
  NvtxRange nvtx("qqa_exchange_emulate");
  if (!hs || G < 1 || G > qqa::kMaxRanks) return fail(QQA_ERR_INVALID_ARG, "handles is NULL or G not in 1..8");
  if (n_steps < 0 || (n_steps > 0 && !gamma_host)) return fail(QQA_ERR_INVALID_ARG, "bad n_steps or gamma NULL");
  for (int r = 0; r < G; ++r) {
    const qqa_handle* h = hs[r];
    if (!h) return fail(QQA_ERR_INVALID_ARG, "a handle is NULL");
    if (!h->xmode || h->xG != G || h->xrank != r)
      return fail(QQA_ERR_INVALID_ARG, "every shard r must have the fused exchange attached as rank r of G");
    if (h->device != hs[0]->device || h->stream != hs[0]->stream || h->s.n != hs[0]->s.n ||
        h->s.lanes != hs[0]->s.lanes || h->s.vpl != hs[0]->s.vpl || h->s.SB != hs[0]->s.SB ||
        step_mode(h->cfg, h->s.weighted) != step_mode(hs[0]->cfg, hs[0]->s.weighted) || h->step != hs[0]->step ||
        h->cur != hs[0]->cur || h->scur != hs[0]->scur || h->xsync != hs[0]->xsync ||
        h->xslotted != hs[0]->xslotted)
      return fail(QQA_ERR_INVALID_ARG, "emulated shards must share device, stream, layout, mode and be in lockstep");
  }
  qqa_handle* h0 = hs[0];
  int st = set_device(h0);
  if (st) return st;
  if (n_steps == 0 || h0->s.n == 0) return QQA_OK;
  const qqa::XEmulKernel ke = qqa::xemul_kernel(h0->s.lanes, h0->s.vpl, step_mode(h0->cfg, h0->s.weighted),
                                                full_lanes(h0->s));
  if (!ke) return fail(QQA_ERR_UNSUPPORTED, "no emulation kernel for this layout / mode");
  // the per-(step, rank) parameters exactly as do_steps_x would launch them, step by step (the handles'
  // step counters advance while they are built; restored if the launch fails)
  struct Saved { int cur, scur; int64_t step, launches; unsigned long long xsync; };
  std::vector<Saved> saved((size_t)G);
  for (int r = 0; r < G; ++r) saved[r] = {hs[r]->cur, hs[r]->scur, hs[r]->step, hs[r]->launches, hs[r]->xsync};
  auto restore = [&](int status) {
    for (int r = 0; r < G; ++r) {
      hs[r]->cur = saved[r].cur; hs[r]->scur = saved[r].scur; hs[r]->step = saved[r].step;
      hs[r]->launches = saved[r].launches; hs[r]->xsync = saved[r].xsync;
    }
    return status;
  };
  std::vector<qqa::StepParams> base((size_t)G);
  std::vector<qqa::StepVar> var((size_t)n_steps * G);
  std::vector<qqa::XParams> xp((size_t)n_steps * G);
  for (int r = 0; r < G; ++r) base[r] = xstep_base(hs[r]);
  for (int64_t k = 0; k < n_steps; ++k)
    for (int r = 0; r < G; ++r) {
      qqa_handle* h = hs[r];
      const int a = h->cur, b = h->cur ^ 1;
      const int sa = h->scur, sb = (h->scur + 1) % 3, sz = (h->scur + 2) % 3;
      var[(size_t)k * G + r] = xstep_var(h, gamma_host[k]);
      xp[(size_t)k * G + r] = make_xparams(h, sa, sb, sz, a, b);
      h->xsync += h->xslotted ? 2 : 1;
      h->cur = b;
      h->scur = sb;
      h->step += 1;
      h->launches++;
    }
  const size_t nb = base.size() * sizeof(qqa::StepParams), nv = var.size() * sizeof(qqa::StepVar),
               nx = xp.size() * sizeof(qqa::XParams);
#define QQA_CUDA_R(call)                                                                          \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return restore(fail(QQA_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  char* d = nullptr;
  QQA_CUDA_R(cudaMalloc(&d, nb + nv + nx + 512));
  struct Free { char* p; ~Free() { cudaFree(p); } } guard{d};
  char* db = d;
  char* dv = d + up(nb, 256);
  char* dx = dv + up(nv, 256);
  QQA_CUDA_R(cudaMemcpyAsync(db, base.data(), nb, cudaMemcpyHostToDevice, h0->stream));
  QQA_CUDA_R(cudaMemcpyAsync(dv, var.data(), nv, cudaMemcpyHostToDevice, h0->stream));
  QQA_CUDA_R(cudaMemcpyAsync(dx, xp.data(), nx, cudaMemcpyHostToDevice, h0->stream));
  int per_sm = 0;
  QQA_CUDA_R(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)ke, 256, 0));
  const int cta_per_rank = std::max(1, per_sm * h0->sm_count / G);
  if ((int64_t)per_sm * h0->sm_count < G) return restore(fail(QQA_ERR_UNSUPPORTED, "too few co-resident CTAs for G ranks"));
  qqa::XEmulParams E{};
  E.base = reinterpret_cast<const qqa::StepParams*>(db);
  E.var = reinterpret_cast<const qqa::StepVar*>(dv);
  E.xp = reinterpret_cast<const qqa::XParams*>(dx);
  E.G = G;
  E.nsteps = (int)n_steps;
  E.cta_per_rank = cta_per_rank;
  E.slotted = h0->xslotted ? 1 : 0;
  void* args[] = {(void*)&E};
  QQA_CUDA_R(cudaLaunchCooperativeKernel((const void*)ke, dim3(G * cta_per_rank), dim3(256), args, 0, h0->stream));
#undef QQA_CUDA_R
  QQA_CUDA(cudaStreamSynchronize(h0->stream));
  return QQA_OK;
}

int qqa_run_linear(qqa_handle* h, float gmin, float gmax, int64_t total_steps, int64_t t0, int64_t t1) {
  NvtxRange nvtx("qqa_run_linear");
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  if (total_steps < 1 || t0 < 0 || t1 < t0 || t1 > total_steps)
    return fail(QQA_ERR_INVALID_ARG, "need 0 <= t0 <= t1 <= total_steps, total_steps >= 1");
  int st = set_device(h);
  if (st) return st;
  std::vector<float> gam((size_t)(t1 - t0));
  for (int64_t t = t0; t < t1; ++t)  // P:245, P:667 (reading R10)
    gam[(size_t)(t - t0)] = (total_steps == 1)
        ? gmin
        : (float)((double)gmin + (((double)gmax - (double)gmin) * (double)t) / (double)(total_steps - 1));
  return do_steps(h, gam.data(), t1 - t0);
}

}  // extern "C"

namespace {

// K3-K5 on the device: round + pack, per-(replica, instance) counts, all-gather of
// the counts over ranks, energies + argmin of the totals and of every instance.
int evaluate_core_kary(qqa_handle* h) {
  const Shape& s = h->s;
  const int off = h->cfg.replica_offset;
  StepKKernel ks;
  InitKKernel ki;
  PackKKernel kp;
  pick_kary(s.KP, s.K, step_mode(h->cfg, h->s.weighted), ks, ki, kp);
  uint8_t* X8 = (uint8_t*)h->X;
  const int64_t ns = (int64_t)s.n * s.S_local;
  if (ns > 0) {  // K3: x = argmax_k P
    kp<<<(int)std::max<int64_t>(1, std::min<int64_t>((ns + 255) / 256, (int64_t)h->sm_count * 16)), 256, 0,
         h->stream>>>(h->p[h->cur], X8, s.n, s.S_local, s.K);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  QQA_CUDA(cudaMemsetAsync(h->counts, 0, 3 * (size_t)s.S_total * sizeof(long long), h->stream));
  unsigned long long* mine = h->counts + 3 * (size_t)off;
  if (s.n > 0) {  // K4: conflicts per replica
    const int W = (s.S_local + 31) / 32;
    const int R = (int)std::max<int64_t>(1, std::min<int64_t>(s.n, (int64_t)h->sm_count * 64 / W));
    const int CH = (s.n + R - 1) / R;
    const int64_t warps = (int64_t)W * R;
    qqa::k_eval_K<<<(int)((warps + 7) / 8), 256, 0, h->stream>>>(h->rowptr, h->colidx, X8, s.n, s.S_local, W, R,
                                                                  CH, mine);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  qqa::k_conflicts_finish<<<1, 256, 0, h->stream>>>((long long*)mine, s.S_local, (long long)(s.nnz / 2));
  QQA_CUDA(cudaGetLastError());
  h->launches++;
  if (h->comm && h->nranks > 1)
    QQA_NCCL(ncclAllGather(mine, h->counts, 3 * (size_t)s.S_local, ncclInt64, h->comm, h->stream));
  qqa::k_argmin<<<1, 1024, 0, h->stream>>>((const long long*)h->counts, 3, s.S_total, qqa::kCOLORING, 0.0,
                                           h->energy, h->best, h->beste, nullptr);
  QQA_CUDA(cudaGetLastError());
  h->launches++;
  QQA_CUDA(cudaMemcpyAsync(h->genergy, h->energy, (size_t)s.S_total * sizeof(double), cudaMemcpyDeviceToDevice,
                           h->stream));
  QQA_CUDA(cudaMemcpyAsync(h->gbest, h->best, sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
  QQA_CUDA(cudaMemcpyAsync(h->gbeste, h->beste, sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  return QQA_OK;
}

// Best replica's x as bytes into xbuf (K-ary: its colours), on the owner rank.
int extract_x(qqa_handle* h, int s_local) {
  const Shape& s = h->s;
  const int blocks = std::max(1, std::min((s.n + 255) / 256, h->sm_count * 4));
  if (s.kary)
    qqa::k_extract_K<<<blocks, 256, 0, h->stream>>>((const uint8_t*)h->X, s.n, s.S_local, s_local, h->xbuf);
  else
    qqa::k_extract<<<blocks, 256, 0, h->stream>>>(h->X, s.n, s.W, s_local, h->xbuf);
  QQA_CUDA(cudaGetLastError());
  h->launches++;
  return QQA_OK;
}

int evaluate_core(qqa_handle* h) {
  if (h->s.kary) return evaluate_core_kary(h);
  const Shape& s = h->s;
  const int off = h->cfg.replica_offset;
  if (s.n > 0) {  // K3: round + pack
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)s.n * s.W * 32 + 255) / 256, (int64_t)h->sm_count * 16));
    const float thr = (h->cfg.map == QQA_MAP_CLAMP) ? 0.5f : 0.0f;   // x = Theta(p - 1/2)
    qqa::k_pack<<<blocks, 256, 0, h->stream>>>(h->theta, h->X, s.n, s.SB, s.S_local, s.W, thr);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  // K4: counts of the local replicas at their global slots, [S_total][G][3]
  QQA_CUDA(cudaMemsetAsync(h->counts, 0, 3 * (size_t)s.S_total * s.G * sizeof(long long), h->stream));
  if (s.weighted) QQA_CUDA(cudaMemsetAsync(h->wsums, 0, 2 * (size_t)s.S_total * sizeof(long long), h->stream));
  if (s.n > 0) {
    const int R = (int)std::max<int64_t>(1, std::min<int64_t>(s.n, (int64_t)h->sm_count * 64 / s.W));
    const int CH = (s.n + R - 1) / R;
    const int64_t warps = (int64_t)s.W * R;
    const int blocks = (int)((warps + 7) / 8);
    qqa::k_eval<<<blocks, 256, 0, h->stream>>>(h->rowptr, h->colidx, h->X, h->gor, s.n, s.W, R, CH, s.S_local, s.G,
                                               h->counts + 3 * (size_t)off * s.G, h->w,
                                               (unsigned long long*)h->wsums + 2 * (size_t)off);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  if (h->cfg.problem == QQA_MAXCLIQUE_SPARSE) {   // original-graph counts -> complement counts (G = 1)
    qqa::k_clique_counts<<<std::max(1, std::min((s.S_local + 255) / 256, h->sm_count)), 256, 0, h->stream>>>(
        (long long*)h->counts + 3 * (size_t)off, s.S_local, (long long)s.n);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  if (h->comm && h->nranks > 1) {
    QQA_NCCL(ncclAllGather(h->counts + 3 * (size_t)off * s.G, h->counts, 3 * (size_t)s.S_local * s.G, ncclInt64,
                           h->comm, h->stream));
    if (s.weighted)
      QQA_NCCL(ncclAllGather(h->wsums + 2 * (size_t)off, h->wsums, 2 * (size_t)s.S_local, ncclInt64, h->comm,
                             h->stream));
  }
  const int prob = h->cfg.problem == QQA_MAXCUT ? qqa::kMAXCUT : qqa::kMIS;   // cliques: complement counts
  const long long* tot = (const long long*)h->counts;
  if (s.G > 1) {  // totals over instances = the energy of the union graph
    qqa::k_sum_groups<<<std::max(1, std::min((3 * s.S_total + 255) / 256, h->sm_count * 4)), 256, 0, h->stream>>>(
        (const long long*)h->counts, s.S_total, s.G, h->tot);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
    tot = h->tot;
    qqa::k_argmin<<<s.G, 1024, 0, h->stream>>>((const long long*)h->counts, 3 * s.G, s.S_total, prob,
                                                (double)h->cfg.penalty, h->genergy, h->gbest, h->gbeste, nullptr);
    QQA_CUDA(cudaGetLastError());
    h->launches++;
  }
  // K5: energies + argmin over all replicas (of the totals)
  qqa::k_argmin<<<1, 1024, 0, h->stream>>>(tot, 3, s.S_total, prob, (double)h->cfg.penalty, h->energy, h->best,
                                           h->beste, s.weighted ? h->wsums : nullptr);
  QQA_CUDA(cudaGetLastError());
  h->launches++;
  if (s.G == 1) {  // the single instance is the whole graph
    QQA_CUDA(cudaMemcpyAsync(h->genergy, h->energy, (size_t)s.S_total * sizeof(double), cudaMemcpyDeviceToDevice,
                             h->stream));
    QQA_CUDA(cudaMemcpyAsync(h->gbest, h->best, sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
    QQA_CUDA(cudaMemcpyAsync(h->gbeste, h->beste, sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  }
  return QQA_OK;
}

int finish_eval(qqa_handle* h) {
  int flag = 0;
  QQA_CUDA(cudaMemcpyAsync(&flag, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  if (h->comm) {
    ncclResult_t async_err = ncclSuccess;
    ncclCommGetAsyncError(h->comm, &async_err);
    if (async_err != ncclSuccess) return fail(QQA_ERR_COMM, ncclGetErrorString(async_err));
  }
  if (flag & 4) return fail(QQA_ERR_COMM, "fused exchange: a peer rank never arrived at a step barrier");
  if (flag & 1) return fail(QQA_ERR_NONFINITE, "a non-finite theta appeared during the run");
  return QQA_OK;
}

}  // namespace

extern "C" {

int qqa_round_evaluate(qqa_handle* h, qqa_replica_result* per_replica, int32_t* best_replica,
                       double* best_energy, uint8_t* best_x) {
  NvtxRange nvtx("qqa_round_evaluate");
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  if ((st = evaluate_core(h))) return st;
  const Shape& s = h->s;
  const int off = h->cfg.replica_offset;
  const long long* tot = (s.G > 1) ? h->tot : (const long long*)h->counts;
  int best = 0;
  double be = 0.0;
  QQA_CUDA(cudaMemcpyAsync(&best, h->best, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  QQA_CUDA(cudaMemcpyAsync(&be, h->beste, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  std::vector<long long> cnt, wsm;
  std::vector<double> en;
  if (per_replica) {
    cnt.resize(3 * (size_t)s.S_local);
    en.resize((size_t)s.S_local);
    if (s.weighted) {
      wsm.resize(2 * (size_t)s.S_local);
      QQA_CUDA(cudaMemcpyAsync(wsm.data(), h->wsums + 2 * (size_t)off, wsm.size() * sizeof(long long),
                               cudaMemcpyDeviceToHost, h->stream));
    }
    QQA_CUDA(cudaMemcpyAsync(cnt.data(), tot + 3 * (size_t)off, cnt.size() * sizeof(long long),
                             cudaMemcpyDeviceToHost, h->stream));
    QQA_CUDA(cudaMemcpyAsync(en.data(), h->energy + off, en.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             h->stream));
  }
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  if (best_x && s.n > 0) {
    const int owner = best / s.S_local;
    if (!h->comm || h->nranks == 1 || owner == h->rank) {
      if ((st = extract_x(h, best - off))) return st;
    }
    if (h->comm && h->nranks > 1) {
      QQA_NCCL(ncclBroadcast(h->xbuf, h->xbuf, (size_t)s.n, ncclUint8, owner, h->comm, h->stream));
    }
    QQA_CUDA(cudaMemcpyAsync(best_x, h->xbuf, (size_t)s.n, cudaMemcpyDeviceToHost, h->stream));
  }
  if ((st = finish_eval(h))) return st;
  if (per_replica) {
    for (int k = 0; k < s.S_local; ++k) {
      qqa_replica_result& r = per_replica[k];
      r.size = cnt[3 * k + 0];
      r.violations = cnt[3 * k + 1];
      r.cut = cnt[3 * k + 2];
      r.energy = en[k];
      r.feasible = (h->cfg.problem == QQA_MAXCUT) ? 1 : (r.violations == 0);   // colouring: proper
      r.replica = off + k;
      r.wviolations = s.weighted ? (double)wsm[2 * k] * 0x1p-24 : (double)r.violations;
      r.wcut = s.weighted ? (double)wsm[2 * k + 1] * 0x1p-24 : (double)r.cut;
    }
  }
  if (best_replica) *best_replica = best;
  if (best_energy) *best_energy = be;
  return QQA_OK;
}

int qqa_n_groups(qqa_handle* h, int32_t* n_groups) {
  if (!h || !n_groups) return fail(QQA_ERR_INVALID_ARG, "handle or n_groups is NULL");
  *n_groups = h->s.G;
  return QQA_OK;
}

int qqa_round_evaluate_groups(qqa_handle* h, int64_t* counts, double* energy, int32_t* best_replica,
                              double* best_energy, uint8_t* best_x) {
  NvtxRange nvtx("qqa_round_evaluate_groups");
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  if ((st = evaluate_core(h))) return st;
  const Shape& s = h->s;
  const int off = h->cfg.replica_offset;
  if (best_replica) QQA_CUDA(cudaMemcpyAsync(best_replica, h->gbest, (size_t)s.G * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  if (best_energy) QQA_CUDA(cudaMemcpyAsync(best_energy, h->gbeste, (size_t)s.G * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  if (energy)  // [G][S_local]: this rank's replicas of every instance
    QQA_CUDA(cudaMemcpy2DAsync(energy, (size_t)s.S_local * sizeof(double), h->genergy + off,
                               (size_t)s.S_total * sizeof(double), (size_t)s.S_local * sizeof(double), (size_t)s.G,
                               cudaMemcpyDeviceToHost, h->stream));
  std::vector<long long> cnt;
  if (counts) {  // device [S_total][G][3] -> host [G][S_local][3]
    cnt.resize(3 * (size_t)s.S_local * s.G);
    QQA_CUDA(cudaMemcpyAsync(cnt.data(), h->counts + 3 * (size_t)off * s.G, cnt.size() * sizeof(long long),
                             cudaMemcpyDeviceToHost, h->stream));
  }
  if (best_x && s.n > 0) {
    if (h->gor) {
      qqa::k_extract_groups<<<std::max(1, std::min((s.n + 255) / 256, h->sm_count * 4)), 256, 0, h->stream>>>(
          h->X, h->gor, h->gbest, s.n, s.W, off, s.S_local, h->xbuf);
      QQA_CUDA(cudaGetLastError());
      h->launches++;
      if (h->comm && h->nranks > 1)  // exactly one rank holds each row's best replica: sum = that value
        QQA_NCCL(ncclAllReduce(h->xbuf, h->xbuf, (size_t)s.n, ncclUint8, ncclSum, h->comm, h->stream));
      QQA_CUDA(cudaMemcpyAsync(best_x, h->xbuf, (size_t)s.n, cudaMemcpyDeviceToHost, h->stream));
    } else {
      int best = 0;
      QQA_CUDA(cudaMemcpyAsync(&best, h->best, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      QQA_CUDA(cudaStreamSynchronize(h->stream));
      const int owner = best / s.S_local;
      if (!h->comm || h->nranks == 1 || owner == h->rank) {
        if ((st = extract_x(h, best - off))) return st;
      }
      if (h->comm && h->nranks > 1)
        QQA_NCCL(ncclBroadcast(h->xbuf, h->xbuf, (size_t)s.n, ncclUint8, owner, h->comm, h->stream));
      QQA_CUDA(cudaMemcpyAsync(best_x, h->xbuf, (size_t)s.n, cudaMemcpyDeviceToHost, h->stream));
    }
  }
  if ((st = finish_eval(h))) return st;
  if (counts)
    for (int k = 0; k < s.S_local; ++k)
      for (int g = 0; g < s.G; ++g)
        for (int c = 0; c < 3; ++c)
          counts[((size_t)g * s.S_local + k) * 3 + c] = cnt[((size_t)k * s.G + g) * 3 + c];
  return QQA_OK;
}

int qqa_get_state(qqa_handle* h, float* theta, float* m, float* v, float* p, int64_t* step) {
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  // K-ary: the parameter is P itself, so theta and p both receive P
  const float* src[4] = {h->s.kary ? h->p[h->cur] : h->theta, h->m, h->v, h->p[h->cur]};
  float* dst[4] = {theta, m, v, p};
  for (int k = 0; k < 4; ++k)
    if (dst[k] && (st = copy_blocked(h, dst[k], const_cast<float*>(src[k]), cudaMemcpyDeviceToHost))) return st;
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  if (step) *step = h->step;
  return QQA_OK;
}

int qqa_get_stats(qqa_handle* h, float* c, int64_t* sumD, int64_t* sumD2) {
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  const size_t n = (size_t)h->s.n * (h->s.kary ? h->s.K : 1);   // statistics entries
  if (c && n) QQA_CUDA(cudaMemcpyAsync(c, h->c[h->cur], n * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  const long long* sums = h->sums[h->scur];
  if (h->xmode && n && (sumD || sumD2)) {   // owner rows hold the totals: gather them into the scratch
    const qqa::XParams X = make_xparams(h, h->scur, h->scur, h->scur, h->cur, h->cur);
    const int blocks = std::max(1, std::min((int)((n + 255) / 256), h->sm_count * 8));
    if (h->xslotted)   // the current statistics are the G writers' slots of parity (step & 1) at each owner
      qqa::k_xs_gather<<<blocks, 256, 0, h->stream>>>(X, (int)n, (int)(h->step & 1), h->ws_sums[2], h->flag);
    else
      qqa::k_x_gather<<<blocks, 256, 0, h->stream>>>(X, (int)n, h->ws_sums[0], h->flag);
    QQA_CUDA(cudaGetLastError());
    sums = h->xslotted ? h->ws_sums[2] : h->ws_sums[0];
  }
  if (sumD && n)
    QQA_CUDA(cudaMemcpyAsync(sumD, sums, n * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  if (sumD2 && n)
    QQA_CUDA(cudaMemcpyAsync(sumD2, sums + n, n * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  int flag = 0;
  if (h->xmode) QQA_CUDA(cudaMemcpyAsync(&flag, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  if (flag & 4) return fail(QQA_ERR_COMM, "fused exchange: a peer rank never arrived at a step barrier");
  return QQA_OK;
}

int qqa_set_state(qqa_handle* h, const float* theta, const float* m, const float* v, const float* c, int64_t step) {
  if (!h || !theta || !m || !v) return fail(QQA_ERR_INVALID_ARG, "handle, theta, m or v is NULL");
  if (step < 0) return fail(QQA_ERR_INVALID_ARG, "step < 0");
  int st = set_device(h);
  if (st) return st;
  const Shape& s = h->s;
  float* param = s.kary ? h->p[0] : h->theta;   // K-ary: the parameter is P (launch_init copies it to p[1])
  const size_t bytes = s.kary ? (size_t)s.n * s.S_local * s.KP * sizeof(float)
                              : ((size_t)s.n + 1) * s.S_p * sizeof(float);
  for (float* buf : {param, h->m, h->v}) QQA_CUDA(cudaMemsetAsync(buf, 0, bytes, h->stream));
  const float* src[3] = {theta, m, v};
  float* dst[3] = {param, h->m, h->v};
  for (int k = 0; k < 3; ++k)
    if ((st = copy_blocked(h, const_cast<float*>(src[k]), dst[k], cudaMemcpyHostToDevice))) return st;
  const float* cdev = nullptr;
  const size_t nk = (size_t)s.n * (s.kary ? s.K : 1);
  if (c && s.n > 0) {
    QQA_CUDA(cudaMemcpyAsync(h->c[1], c, nk * sizeof(float), cudaMemcpyHostToDevice, h->stream));
    cdev = h->c[1];
  }
  if ((st = launch_init(h, true, cdev))) return st;
  h->step = step;
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  return QQA_OK;
}

int qqa_profile(qqa_handle* h, int enable) {
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  h->profiling = enable != 0;
  h->ev_used = 0;
  h->prof_launches = 0;
  h->prof_ms = 0.0;
  return QQA_OK;
}

int qqa_profile_read(qqa_handle* h, double* step_kernel_ms, int64_t* step_launches) {
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  int st = set_device(h);
  if (st) return st;
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  double total = h->prof_ms;
  for (size_t k = 0; k + 1 < h->ev_used; k += 2) {
    float ms = 0.f;
    QQA_CUDA(cudaEventElapsedTime(&ms, h->ev[k], h->ev[k + 1]));
    total += ms;
  }
  h->prof_ms = total;
  h->ev_used = 0;
  if (step_kernel_ms) *step_kernel_ms = total;
  if (step_launches) *step_launches = h->prof_launches;
  return QQA_OK;
}

int qqa_launch_count(qqa_handle* h, int64_t* launches) {
  if (!h || !launches) return fail(QQA_ERR_INVALID_ARG, "handle or launches is NULL");
  *launches = h->launches;
  return QQA_OK;
}

}  // extern "C"

namespace {
// Exchange buffer of one rank: atomics mode: sums [3][2][n]; slotted mode: slots [2][G][2][ceil(n/G)] then
// totals [2][ceil(n/G)] (at most 48 n + 4 KB bytes for G <= 8); the arrival counter and ticket after both.
size_t xflag_offset(const qqa_handle* h) { return 6 * (size_t)h->s.n * sizeof(long long) + 4096; }
}  // namespace

extern "C" {

int qqa_exchange_bytes(qqa_handle* h, size_t* bytes) {
  if (!h || !bytes) return fail(QQA_ERR_INVALID_ARG, "handle or bytes is NULL");
  *bytes = xflag_offset(h) + 256;   // statistics region, then the arrival counter and ticket
  return QQA_OK;
}

int qqa_attach_exchange(qqa_handle* h, const uint64_t* peer_bufs, int rank, int nranks) {
  return qqa_attach_exchange_mode(h, peer_bufs, rank, nranks, QQA_EXCHANGE_ATOMIC);
}

int qqa_attach_exchange_mode(qqa_handle* h, const uint64_t* peer_bufs, int rank, int nranks, int mode) {
  if (!h || !peer_bufs) return fail(QQA_ERR_INVALID_ARG, "handle or peer_bufs is NULL");
  if (mode != QQA_EXCHANGE_ATOMIC && mode != QQA_EXCHANGE_SLOTTED) return fail(QQA_ERR_INVALID_ARG, "unknown exchange mode");
  if (nranks < 1 || nranks > qqa::kMaxRanks || rank < 0 || rank >= nranks)
    return fail(QQA_ERR_INVALID_ARG, "need 1 <= nranks <= 8 and 0 <= rank < nranks");
  if (h->s.kary || (step_mode(h->cfg, h->s.weighted) & qqa::kModeSparseClique))
    return fail(QQA_ERR_UNSUPPORTED, "the fused exchange supports the binary problems except the printed clique");
  if ((int64_t)h->s.S_local * nranks != h->s.S_total || h->cfg.replica_offset != rank * h->s.S_local)
    return fail(QQA_ERR_INVALID_ARG, "sharding must be S_total = nranks * S_local and replica_offset = rank * S_local");
  if (h->comm && (h->rank != rank || h->nranks != nranks))
    return fail(QQA_ERR_INVALID_ARG, "rank / nranks differ from the attached communicator");
  const bool slotted = mode == QQA_EXCHANGE_SLOTTED;
  const int smode = step_mode(h->cfg, h->s.weighted);
  if (!pick_xstep(h->s.lanes, h->s.vpl, smode, full_lanes(h->s)))
    return fail(QQA_ERR_UNSUPPORTED, "no fused-exchange kernel for this replica layout");
  const qqa::XStepKernel kxs = slotted ? pick_xsstep(h->s.lanes, h->s.vpl, smode, full_lanes(h->s)) : nullptr;
  if (slotted && (h->s.B != 1 || !kxs))
    return fail(QQA_ERR_UNSUPPORTED, "the owner-slotted exchange needs one replica block (S_local <= 32 per 128 MB)");
  int st = set_device(h);
  if (st) return st;
  int grid_xs = 0;
  if (slotted) {   // cooperative launch: every CTA of the step kernel resident (the mid-kernel barrier)
    int per_sm = 0, coop = 0;
    QQA_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device));
    QQA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kxs, 256, 0));
    if (!coop || per_sm < 1) return fail(QQA_ERR_UNSUPPORTED, "no cooperative launch for the owner-slotted exchange");
    const int need = (int)std::max<int64_t>(1, ((int64_t)h->s.n * h->s.lanes + 255) / 256);
    grid_xs = std::max(1, std::min(need, per_sm * h->sm_count));
  }
  const size_t n2 = 2 * (size_t)h->s.n;
  for (int r = 0; r < nranks; ++r) {
    if (!peer_bufs[r] || peer_bufs[r] % 256) return fail(QQA_ERR_INVALID_ARG, "peer buffer NULL or not 256-byte aligned");
    long long* base = reinterpret_cast<long long*>(peer_bufs[r]);
    h->xbase[r] = base;
    for (int k = 0; k < 3; ++k) h->xsums[r][k] = base + k * n2;
    h->xflag[r] = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + xflag_offset(h));
  }
  if (!h->xmode)
    for (int k = 0; k < 3; ++k) h->ws_sums[k] = h->sums[k];
  h->xticket = reinterpret_cast<unsigned int*>(h->xflag[rank] + 1);
  QQA_CUDA(cudaMemsetAsync(h->xbase[rank], 0, xflag_offset(h) + 256, h->stream));
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  if (slotted) {   // the handle's own buffers keep the local partials (init); the exchange lives in the slots
    for (int k = 0; k < 3; ++k) h->sums[k] = h->ws_sums[k];
    if (h->comm) {  // every rank's buffer is zeroed before any rank scatters into it: a collective in between
      QQA_NCCL(ncclAllReduce(h->best, h->best, 1, ncclInt32, ncclSum, h->comm, h->stream));
    }
    h->xdefer_init = (h->comm == nullptr);   // emulated shards: qqa_loopback_sync_init scatters and arrives
  } else {
    for (int k = 0; k < 3; ++k) h->sums[k] = h->xsums[rank][k];
    h->xdefer_init = false;
  }
  h->xslotted = slotted;
  h->grid_xs = grid_xs;
  h->xmode = true;
  h->xrank = rank;
  h->xG = nranks;
  h->xsync = 0;
  h->comm_chunks = 1;
  h->step = 0;
  // re-initialise into the exchange buffers; with a communicator the all-reduced totals end with the
  // first barrier arrival, without one (emulated shards) qqa_loopback_sync_init completes them
  if ((st = launch_init(h, false, nullptr))) return st;
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  return QQA_OK;
}

int qqa_detach_exchange(qqa_handle* h) {
  if (!h) return fail(QQA_ERR_INVALID_ARG, "handle is NULL");
  if (!h->xmode) return QQA_OK;
  int st = set_device(h);
  if (st) return st;
  QQA_CUDA(cudaStreamSynchronize(h->stream));
  for (int k = 0; k < 3; ++k) h->sums[k] = h->ws_sums[k];   // the workspace's own statistic buffers again
  for (int r = 0; r < qqa::kMaxRanks; ++r) {
    for (int k = 0; k < 3; ++k) h->xsums[r][k] = nullptr;
    h->xflag[r] = nullptr;
  }
  h->xticket = nullptr;
  for (int r = 0; r < qqa::kMaxRanks; ++r) h->xbase[r] = nullptr;
  h->xslotted = false;
  h->xdefer_init = false;
  h->xmode = false;
  h->xrank = 0;
  h->xG = 1;
  h->xsync = 0;
  if ((st = setup_overlap(h))) return st;
  return QQA_OK;   // the replica state must be re-initialised (qqa_reset / qqa_set_state, collective) before a run
}

int qqa_step_path(qqa_handle* h, int* path) {
  if (!h || !path) return fail(QQA_ERR_INVALID_ARG, "handle or path is NULL");
  *path = h->s.kary ? QQA_PATH_KARY : h->xmode ? QQA_PATH_EXCHANGE : use_cluster(h, 2) ? QQA_PATH_CLUSTER
                                    : use_persistent(h, 2) ? QQA_PATH_PERSISTENT : QQA_PATH_STEP;
  return QQA_OK;
}

int qqa_replica_block(qqa_handle* h, int* SB) {
  if (!h || !SB) return fail(QQA_ERR_INVALID_ARG, "handle or SB is NULL");
  *SB = h->s.kary ? 0 : h->s.SB;
  return QQA_OK;
}

int qqa_destroy(qqa_handle* h) {
  if (!h) return QQA_OK;
  int st = set_device(h);
  if (st) return st;
  cudaStreamSynchronize(h->stream);
  h->comm = nullptr;
  h->comm_box.reset();   // destroys the communicator when no other handle shares it
  for (cudaEvent_t e : h->chunk_ev) cudaEventDestroy(e);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  delete h;
  return QQA_OK;
}

}  // extern "C"
