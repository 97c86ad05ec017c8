/*
 * qqa.h -- C ABI of libqqa.so: the data-parallel hot path of Parallel
 * Quasi-Quantum Annealing (PQQA, arXiv 2409.02135) on NVIDIA B200 (sm_100a).
 *
 * "P:nnn" cites a line of the paper's text. The path, per step and
 * per replica s of the S parallel runs:
 *
 *   p      = sigmoid(theta)                                    P:143 (north_star)
 *   q_i    = sum_{j in N(i)} p_j                               CSR gather
 *   dR/dp  = dl/dp + gamma * ds/dp - alpha_c (p - mu_i)/STD_i   Eq. 6, 7, 10
 *            (evaluated as (p - mu_i) kc_i, kc_i = -alpha_c / STD_i once per row)
 *            MIS / max-clique-on-complement: dl/dp = -1 + lambda q
 *            Max-Cut:                        dl/dp = -deg + 2 q
 *            ds/dp = -2 alpha (2p - 1)^(alpha - 1)                     (Eq. 7)
 *   theta  <- AdamW(theta, dR/dp * p (1 - p))
 *            (+ sqrt(2 lr T) xi when temperature T > 0)        Eq. 9
 *   gamma  linear from gamma_min to gamma_max
 *   x      = Theta(p - 1/2)  (theta >= 0, Theta(0) = 1)
 *
 * With map = QQA_MAP_CLAMP (the paper's experimental setting, "sensitive
 * transitions", Eq. 11) the parameter is p itself:
 *   p' = AdamW(p, dR/dp) (+ sqrt(2 lr T) xi);  p = Clamp(p') into [0, 1];
 *   x = Theta(p - 1/2) evaluated as p >= 1/2; p_0 = 1/2 + U(init_lo, init_hi).
 *   energy = -size + lambda * violations  |  -cut
 *   best   = argmin energy (lowest global replica on ties)
 *
 * Every floating-point result follows the fp32 arithmetic contract written in
 * DESIGN.md §3 (fixed IEEE operation order, fixed-point int64 replica stats),
 * so results are bit-identical to the reference oracle and independent of the
 * number of GPUs the replicas are sharded over.
 *
 * CONVENTIONS
 *  - Every function returns a qqa_status (0 = OK) and never aborts; the
 *    thread-local qqa_last_error() describes the last failure.
 *  - All device work is enqueued on the caller's CUDA stream given at create.
 *    Functions marked (sync) synchronise that stream before returning.
 *    Asynchronous failures (non-finite values, NCCL errors) are reported by
 *    the next (sync) call.
 *  - Host pointers are only read/written during the call. The device
 *    workspace belongs to the caller and must outlive the handle.
 *  - Layout of all replica-state arrays crossing this ABI: row-major
 *    [n][S_local] float32 (variable-major, replica-contiguous), no padding.
 */
#ifndef QQA_H_
#define QQA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QQA_ABI_VERSION 9

#if defined(__GNUC__)
#define QQA_API __attribute__((visibility("default")))
#else
#define QQA_API
#endif

typedef enum {
  QQA_OK = 0,
  QQA_ERR_INVALID_ARG = 1,   /* bad sizes / hyper-parameters / null pointers          */
  QQA_ERR_BAD_GRAPH = 2,     /* CSR not symmetric, unsorted, duplicate, loop, range    */
  QQA_ERR_CUDA = 3,          /* CUDA runtime failure (incl. no device)                 */
  QQA_ERR_COMM = 4,          /* NCCL failure                                           */
  QQA_ERR_NONFINITE = 5,     /* a non-finite theta appeared (SPEC.md:396 abort)        */
  QQA_ERR_UNSUPPORTED = 6,   /* valid input outside what this build implements         */
  QQA_ERR_WORKSPACE = 7      /* workspace null, misaligned or too small                */
} qqa_status;

typedef enum {
  QQA_MAP_SIGMOID = 0,  /* p = sigmoid(theta), AdamW on theta (north_star)              */
  QQA_MAP_CLAMP = 1     /* AdamW on p, then Clamp into [0, 1] (Eq. 11)        */
} qqa_map;

typedef enum {
  QQA_MIS = 0,        /* maximum independent set, l = -1^T x + lambda x^T A x / 2       */
  QQA_MAXCUT = 1,     /* max cut, l = -sum_{(i,j) in E} (1 - (2x_i-1)(2x_j-1))/2       */
  QQA_MAXCLIQUE = 2,  /* max clique, solved as MIS on the complement graph (the library
                         builds the complement on the host at create; n <= 65536)                */
  QQA_MAXCLIQUE_SPARSE = 4,  /* max clique with the relaxation exactly as printed at P:715, on the
                         ORIGINAL graph: dl/dp_i = -1 + lambda((T - 1/2) - sum_{j in N(i)} p_j), T =
                         sum_k p_k per replica (exact fixed-point column sums). No complement, so no
                         n limit; at binary x the energy equals QQA_MAXCLIQUE's; counts are reported
                         for the complement as QQA_MAXCLIQUE does. No batches.                 */
  QQA_COLORING = 3    /* graph colouring with K = n_colors colours (NEXT-4, App. B):
                         every variable is a row of K probabilities, s_K entropy, map
                         Clamp-then-normalise, AdamW on the probabilities with the
                         gradient through the map (kary_grad),
                         x = argmax_k, energy = #{(i<j) in E : x_i = x_j}. The
                         map field is ignored; state arrays are [n][S_local][K]; no batches */
} qqa_problem;

/* Hyper-parameters and the replica shard of this process. Copied at create. */
typedef struct {
  int32_t problem;        /* qqa_problem                                                    */
  int32_t alpha;          /* alpha-entropy exponent, even, 2..16 (Eq. 7)                   */
  float penalty;          /* lambda (2); ignored for Max-Cut                        */
  float comm;             /* alpha_c >= 0, communication strength (Eq. 10)                 */
  float lr, beta1, beta2, eps, weight_decay;   /* AdamW                     */
  float init_lo, init_hi; /* theta_0 ~ U(init_lo, init_hi) by a counter hash of
                             (seed, variable, global replica)                              */
  uint64_t seed;
  int32_t S_total;        /* replicas over all ranks (S of Eq. 10), 1..2^20                */
  int32_t replica_offset; /* first global replica held here                                */
  int32_t S_local;        /* replicas held here, 1..1024                                   */
  int32_t map;            /* qqa_map                                                        */
  float temperature;      /* Langevin T >= 0 (0.001); 0 = no noise. xi ~ N(0,1) is a
                             counter-based Box-Muller draw keyed (seed, Adam step, variable,
                             global replica): identical for every sharding               */
  int32_t n_colors;       /* K, 2..16, for QQA_COLORING (ignored otherwise)                 */
  int32_t kary_grad;      /* QQA_COLORING: 1 = the gradient through the Clamp-normalise map,
                             g_k - sum_k' g_k' p_k' (reading R33: the chain rule at W = P, which
                             reproduces Table 4 on the small queens graphs); 0 = dR/dP itself
                             (reading R29). Ignored for the binary problems              */
} qqa_config;

/* Undirected simple graph as symmetric CSR, host memory, copied at create.
 * rowptr[n+1] (rowptr[0] = 0, non-decreasing, rowptr[n] = nnz), colidx[nnz]
 * strictly ascending within each row, no self-loops, (i,j) present iff (j,i).
 *
 * Batch of instances (NEXT-3; "batch parallel computation for multiple
 * ... instances {C_mu}"): the graph is the block-diagonal union of the
 * instances, group_of_row[i] = instance of row i, non-decreasing (each instance
 * is a contiguous row range), in [0, n_groups); no edge may join two instances
 * (QQA_ERR_BAD_GRAPH). The replicas of every instance anneal together in one
 * step kernel; qqa_round_evaluate_groups reports every instance separately.
 * Max clique takes the complement inside each instance. group_of_row = NULL:
 * one instance (n_groups ignored). */
typedef struct {
  int32_t n;
  int64_t nnz;            /* < 2^31 in this build                                          */
  const int64_t* rowptr;
  const int32_t* colidx;
  const int32_t* group_of_row;  /* [n] or NULL                                             */
  int32_t n_groups;             /* 1..2^24 when group_of_row is set                        */
  const float* weights;         /* [nnz] symmetric edge weights (w_ij = w_ji bitwise, finite) or
                                   NULL. P:687: A_ij is the edge weight. MIS: penalty
                                   lambda sum_{(i,j)} w_ij x_i x_j; Max-Cut: cut weight. q_i =
                                   sum_j w_ij p_j as fl(q + fl(w p)) in CSR order. MIS and
                                   Max-Cut only, no batches (QQA_ERR_UNSUPPORTED otherwise) */
} qqa_graph;

/* Evaluation of one rounded replica (integer counts: bit-exact, order-free).
 * QQA_COLORING: size = 0, violations = conflicts #{(i<j) in E : x_i = x_j},
 * cut = |E| - conflicts, energy = conflicts, feasible = (conflicts == 0). */
typedef struct {
  int64_t size;           /* sum_i x_i                                                     */
  int64_t violations;     /* #{(i<j) in E' : x_i = x_j = 1}, E' = E (complement for clique) */
  int64_t cut;            /* #{(i<j) in E' : x_i != x_j}                                   */
  double energy;          /* -size + lambda*violations (MIS, clique) or -cut (Max-Cut)     */
  int32_t feasible;       /* violations == 0 (always 1 for Max-Cut)                        */
  int32_t replica;        /* global replica index                                          */
  double wviolations;     /* weight sum of the violated edges (= violations unweighted),
                             exact: sum of rint(w 2^24) 2^-24                              */
  double wcut;            /* weight sum of the cut edges (= cut unweighted)                 */
} qqa_replica_result;

typedef struct qqa_handle qqa_handle;

QQA_API int qqa_version(void);                          /* QQA_ABI_VERSION                          */
QQA_API const char* qqa_last_error(void);               /* thread-local message of the last failure */
QQA_API const char* qqa_status_string(int status);

/* Device bytes the workspace must have for (graph, config): the replica state theta / m / v / p x 2
 * ([B][n+1][SB] float32), the padded CSR, the statistics and evaluation buffers (and,
 * with the opt-in segmented gather QQA_SEGMENTS=KS, the KS segment CSRs). The layout environment
 * (QQA_BLOCK_REPLICAS, QQA_SEGMENTS) is read here and at qqa_create: it must be the same for both calls
 * (otherwise qqa_create reports WORKSPACE). Host-only; INVALID_ARG / UNSUPPORTED as qqa_create. */
QQA_API int qqa_workspace_bytes(const qqa_graph* g, const qqa_config* cfg, size_t* bytes);

/* Validate and copy the graph, carve the workspace, initialise the replicas: the S parallel runs
 * of P:189-201 (Eq. 8-10), theta_0 ~ U(init_lo, init_hi) (BASELINE.json configs; the paper is silent,
 * reading R18), m = v = 0 (Adam), p_0 = sigma(theta_0) and the replica statistics
 * mu_i, STD_i of Eq. 10. Graph: host pointers, copied (the dense max clique builds the
 * complement on the host). d_workspace: device pointer, 256-byte aligned,
 * >= qqa_workspace_bytes, owned by the caller. stream: cudaStream_t (NULL = legacy default stream).
 * Errors: INVALID_ARG (config / pointers), BAD_GRAPH (the CSR conditions above, checked on the
 * device, or on the host for QQA_MAXCLIQUE), UNSUPPORTED (sizes), WORKSPACE, CUDA. (sync) */
QQA_API int qqa_create(qqa_handle** out, const qqa_graph* g, const qqa_config* cfg,
               void* d_workspace, size_t workspace_bytes, void* stream);

/* Re-initialise the replica state from the seed (as at create: theta_0, m = v = 0, statistics of
 * p_0); step counter 0. With a communicator attached this is collective. Async. */
QQA_API int qqa_reset(qqa_handle* h);

/* Multi-GPU (one process per GPU, replicas sharded: rank r holds
 * [replica_offset, replica_offset + S_local), S_local equal on all ranks). The S parallel runs of
 * P:189-201 interact only through mu_i and STD_i of Eq. 10, so the only exchange is the
 * sum of their fixed-point terms ("batch parallel computation", "additional GPUs").
 * Rank 0 calls qqa_nccl_unique_id and broadcasts the 128 bytes; every rank
 * then calls qqa_attach_comm (collective), which re-initialises the replica
 * state as qqa_reset does (theta_0 depends only on the global replica index,
 * so every sharding starts from the same ensemble). Each step then
 * all-reduces the 2n int64 statistic sums over NCCL. (sync) */
QQA_API int qqa_nccl_unique_id(uint8_t out[128]);   /* host 128 bytes out; COMM on NCCL failure        */
/* id: rank 0's 128 bytes; requires S_total = nranks * S_local and replica_offset = rank * S_local
 * (INVALID_ARG otherwise); the library owns the communicator. COMM on NCCL failure. (sync) */
QQA_API int qqa_attach_comm(qqa_handle* h, const uint8_t id[128], int rank, int nranks);
/* Use donor's communicator (same device, same rank layout) instead of creating
 * one: a handle for a new input can join a running job without another NCCL
 * bootstrap. The communicator lives until the last handle using it is
 * destroyed. Re-initialises h's replica state like qqa_attach_comm. Collective
 * over the donor's ranks. (sync) */
QQA_API int qqa_share_comm(qqa_handle* h, qqa_handle* donor);

/* Loopback exchange (emulation and testing of the sharded path on ONE GPU): G handles hs[r]
 * created with S_total = G S_local and replica_offset = r S_local, no communicator, on one device
 * and one stream. qqa_loopback_sync_init adds their initial statistic sums (call after create /
 * reset / set_state); qqa_loopback_run then runs n_steps in lockstep, adding the int64 sums of all
 * shards after every step -- exactly the per-step NCCL all-reduce -- so the shards reproduce one
 * handle holding all S_total replicas bit for bit. No kernel waits on another. (sync) */
/* Fused statistics exchange over peer memory, replacing the per-step NCCL all-reduce
 * of Eq. 10's sums: rank r owns rows [r ceil(n/G), (r+1) ceil(n/G)) of the int64 sums; each step
 * kernel adds its replicas' terms of row i directly into the OWNER's buffer (atomics at the owner,
 * over NVLink, issued as rows complete) and reads row i's total from the owner at the next step;
 * step boundaries are an arrival-counter barrier in the same buffers. Bit-identical to the NCCL
 * path (exact integer sums).
 *   qqa_exchange_bytes: size of one rank's exchange buffer (device memory, 256-byte aligned, caller-
 *     owned, e.g. torch symmetric memory), identical on every rank.
 *   qqa_attach_exchange: peer_bufs[r] = rank r's exchange buffer as mapped in THIS process (its own
 *     at r = rank); every rank calls it (collectively when a communicator is attached, which stays
 *     in use for init and evaluation). Zeroes this rank's buffer and re-initialises the replicas.
 *     Without a communicator (shards emulated on one device) call qqa_loopback_sync_init next.
 *   Supported: the binary problems, weighted or not, except the printed clique (else UNSUPPORTED). A peer
 *   that never arrives is reported as QQA_ERR_COMM at the next synchronising call (no hang). */
QQA_API int qqa_exchange_bytes(qqa_handle* h, size_t* bytes);
QQA_API int qqa_attach_exchange(qqa_handle* h, const uint64_t* peer_bufs, int rank, int nranks);
/* The same with a choice of exchange: QQA_EXCHANGE_ATOMIC (each rank adds its partials into the owner's rows
 * with remote int64 atomics, one barrier per step) or QQA_EXCHANGE_SLOTTED (each rank STORES its partials into
 * its own slot at the owner -- coalesced plain stores, no remote atomics; after a barrier the owner sums the G
 * slots of its rows, after a second barrier every rank reads the totals; one cooperative step launch with both
 * barriers; needs one replica block). Both bit-identical to the NCCL path. INVALID_ARG / UNSUPPORTED as above.
 * (sync) */
enum { QQA_EXCHANGE_ATOMIC = 0, QQA_EXCHANGE_SLOTTED = 1 };
QQA_API int qqa_attach_exchange_mode(qqa_handle* h, const uint64_t* peer_bufs, int rank, int nranks, int mode);
/* Back from the fused exchange to the NCCL all-reduce path (the handle's own statistic buffers; the peer
 * buffers are no longer touched). Local, no collective; the replica state must then be re-initialised with
 * qqa_reset or qqa_set_state (collective with a communicator) before the next run. No-op without an
 * attached exchange. (sync) */
QQA_API int qqa_detach_exchange(qqa_handle* h);
QQA_API int qqa_loopback_sync_init(qqa_handle** hs, int G);
QQA_API int qqa_loopback_run(qqa_handle** hs, int G, const float* gamma_host, int64_t n_steps);
/* Concurrent one-GPU emulation of the fused exchange (test of its barrier / atomics protocol; DESIGN.md
 * §6): hs[r] = shard r of G (1..8) with qqa_attach_exchange done as rank r of G on one device and stream
 * (buffers on that device), in lockstep after qqa_loopback_sync_init. Runs n_steps steps (gamma_host
 * float[n_steps]) of all G ranks as ONE cooperative launch whose grid is G slices of co-resident CTAs,
 * slice r executing rank r's k_step_x body: the ranks really run at the same time and wait on each
 * other's arrivals (B200_PROFILING.md: ranks that wait on one another must not be separate launches on
 * one GPU). Same results as the per-step k_step_x launches. INVALID_ARG if the shards are not such a
 * set, UNSUPPORTED for layouts without an emulation kernel (lanes > 8 or vpl > 1). (sync) */
QQA_API int qqa_exchange_emulate(qqa_handle** hs, int G, const float* gamma_host, int64_t n_steps);

/* Run n_steps annealing steps (Eq. 6-10 gradient, AdamW P:220-222, sigma / Clamp map P:143 /
 * Eq. 11) with the given per-step gamma (host float[n_steps], read during the call; P:245 the
 * annealing of gamma). The Adam step counter persists across calls (reading R11). Non-finite values
 * surface as NONFINITE at the next (sync) evaluation. INVALID_ARG: n_steps < 0 or gamma NULL. Async. */
QQA_API int qqa_run(qqa_handle* h, const float* gamma_host, int64_t n_steps);

/* Run steps t0..t1-1 of the linear schedule gamma_t = gmin + (gmax-gmin) t/(T-1)
 * over total_steps = T; T = 1 gives gmin. Async. */
QQA_API int qqa_run_linear(qqa_handle* h, float gmin, float gmax, int64_t total_steps, int64_t t0, int64_t t1);

/* Round, evaluate every replica, pick the best over all ranks. For a
 * batch the counts and energies are summed over the instances (the energy of
 * the union graph).
 * per_replica: host [S_local] or NULL; best_x: host uint8[n] (the best replica's
 * x on every rank) or NULL. Returns QQA_ERR_NONFINITE if any step produced a
 * non-finite theta. (sync) */
QQA_API int qqa_round_evaluate(qqa_handle* h, qqa_replica_result* per_replica,
                       int32_t* best_replica, double* best_energy, uint8_t* best_x);

/* Per-instance evaluation of a batch (NEXT-3): round, count and pick,
 * for every instance g, the best replica over all ranks (argmin of the
 * instance's energy, lowest global replica on ties). Host outputs, NULL to skip:
 * counts int64 [n_groups][S_local][3] (size, violations, cut of this rank's
 * replicas), energy double [n_groups][S_local], best_replica int32 [n_groups]
 * (global index), best_energy double [n_groups], best_x uint8 [n] (row i = x of
 * its instance's best replica, on every rank). Without group_of_row this is the
 * single-instance evaluation (n_groups = 1). (sync) */
QQA_API int qqa_round_evaluate_groups(qqa_handle* h, int64_t* counts, double* energy, int32_t* best_replica,
                                      double* best_energy, uint8_t* best_x);
/* Number of instances of the handle's graph (1 without group_of_row). Host-only. */
QQA_API int qqa_n_groups(qqa_handle* h, int32_t* n_groups);

/* Checkpoint / inspection (SURVEY.md §5 checkpoint / resume): host [n][S_local] float arrays
 * (variable-major, replica-contiguous, caller-owned), NULL to skip. theta / m / v: the AdamW state of
 * P:220-222; p = sigmoid(theta) as used by the next step; step = Adam steps taken. (sync)
 * QQA_COLORING: arrays are [n][S_local][K]; theta and p both receive P. */
QQA_API int qqa_get_state(qqa_handle* h, float* theta, float* m, float* v, float* p, int64_t* step);
/* Replica statistics of the current p (Eq. 10): c (shift, float[n]) and the int64 sums
 * (sumD, sumD2: int64[n], already reduced over ranks; fixed point 2^40 of p - c and (p - c)^2).
 * With the fused exchange it waits for the barrier that ends the last step (COMM if a peer never
 * arrived). (sync)
 * QQA_COLORING: per (variable, colour), arrays [n][K]. */
QQA_API int qqa_get_stats(qqa_handle* h, float* c, int64_t* sumD, int64_t* sumD2);
/* Resume from a checkpoint: theta/m/v host [n][S_local] (the AdamW state of P:220-222); c = shift
 * of the statistics (float[n], NULL = 1/2); step = Adam steps taken (reading R11). Recomputes p and
 * the statistics of Eq. 10 from theta. Collective with a communicator. INVALID_ARG on NULL / step < 0. (sync) QQA_COLORING: theta = P, [n][S_local][K]; c [n][K] (NULL = 1/K). */
QQA_API int qqa_set_state(qqa_handle* h, const float* theta, const float* m, const float* v,
                  const float* c, int64_t step);

/* Time every step-kernel launch with CUDA events on the handle's stream. */
QQA_API int qqa_profile(qqa_handle* h, int enable);
/* Sum of step-kernel durations (ms) and launch count since enable. (sync) */
QQA_API int qqa_profile_read(qqa_handle* h, double* step_kernel_ms, int64_t* step_launches);

/* Kernels launched by this handle since create (all kinds). Host-only. */
QQA_API int qqa_launch_count(qqa_handle* h, int64_t* launches);

/* Which step kernel a qqa_run of >= 2 steps uses (fixed at create / attach). Host-only.
 *   QQA_PATH_STEP        one k_finalize + k_step launch per annealing step
 *   QQA_PATH_PERSISTENT  k_run: one cooperative launch per <= 4096 steps (one GPU, p in L2)
 *   QQA_PATH_KARY        k_step_K (graph colouring)
 *   QQA_PATH_EXCHANGE    k_step_x: sharded replicas with the fused statistics exchange (qqa_attach_exchange)
 *   QQA_PATH_CLUSTER     k_run_cluster: the whole anneal in one thread-block cluster's shared memory
 *                        (one GPU, n * S_p <= 32768 and padded nnz * S_p <= 2^19) */
enum { QQA_PATH_STEP = 0, QQA_PATH_PERSISTENT = 1, QQA_PATH_KARY = 2, QQA_PATH_CLUSTER = 3, QQA_PATH_EXCHANGE = 4 };
QQA_API int qqa_step_path(qqa_handle* h, int* path);
/* Replica block SB of the layout [B][n+1][SB] (0 for colouring). Host-only. */
QQA_API int qqa_replica_block(qqa_handle* h, int* SB);

/* Free the handle (and its communicator when no other handle shares it); the workspace is the
 * caller's and is not freed. NULL is OK. (sync) */
QQA_API int qqa_destroy(qqa_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* QQA_H_ */
