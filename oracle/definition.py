"""QQA oracle, fp64 DEFINITION mode.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module. The product path
(``paper_2409_02135_b200``) never does.

Plain fp64 numpy, written equation by equation from PAPER.md (cited as P:<line>):

  * relaxed objectives (Appendix D):  MIS  l = -c^T x + lambda x^T A x / 2
                                      Max-Cut l = -sum_{(i,j) in E} A_ij (1-(2x_i-1)(2x_j-1))/2
                                      max clique = MIS on the complement graph (reading R14)
  * alpha-entropy s(p) = sum_i 1 - (2 p_i - 1)^alpha                          (Eq. 7)
  * QQA objective r = l(p) + gamma s(p)                                       (Eq. 6)
  * ensemble objective R = sum_s r_s - S alpha_c sum_i STD_i, population STD  (Eq. 10)
  * p = sigmoid(theta)                                                        (BASELINE.json north_star)
  * or the sensitive transition with Clamp: AdamW on p, p <- Clamp(p')        (Eq. 11)
  * Langevin noise + sqrt(2 eta T) xi, eta = lr, after the optimizer step     (Eq. 9 / 11)
  * AdamW (decoupled weight decay)
  * gamma linear from gamma_min to gamma_max over the steps
  * rounding x = Theta(p - 1/2)  (evaluated as theta >= 0, Theta(0) = 1)
  * K-ary / graph colouring (NEXT-4): s_K entropy, Clamp-normalise map, AdamW on P (App. B, P:613-647;
    P:672-676; colouring energy P:745-750)

Every function here is pinned by ``tests/test_oracle_definition.py`` against
things other than itself: SPEC.md worked values, central finite differences,
closed forms (Prop. A.2, Theorem 1 limits), and brute force on tiny graphs.
"""
from __future__ import annotations

import itertools

import numpy as np

MIS, MAXCUT, MAXCLIQUE = 0, 1, 2
MAXCLIQUE_SPARSE = 4   # the printed max-clique relaxation on the original graph (NEXT-3 option)
PROBLEM_IDS = {"mis": MIS, "maxcut": MAXCUT, "maxclique": MAXCLIQUE, "maxclique_sparse": MAXCLIQUE_SPARSE}

# STD below this is treated as a non-differentiable point: comm gradient 0
# (reading R6; 0 lies in the subgradient set of sqrt at 0).
STD_FLOOR = 1e-6


def _pid(problem) -> int:
    return PROBLEM_IDS[problem] if isinstance(problem, str) else int(problem)


# --------------------------------------------------------------- graphs
def dense_adjacency(n: int, rowptr, colidx, weights=None) -> np.ndarray:
    """Dense A; with weights, A_ij is the edge weight."""
    A = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for e in range(int(rowptr[i]), int(rowptr[i + 1])):
            A[i, int(colidx[e])] = 1.0 if weights is None else float(weights[e])
    return A


def weighted_sums(A: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Per replica [S][2]: (sum of w_ij over edges (i<j) with x_i = x_j = 1, sum over edges with x_i != x_j)."""
    iu, ju = np.nonzero(np.triu(A != 0, 1))
    w = A[iu, ju][:, None]
    X = X.astype(np.int64)
    return np.stack([(w * (X[iu] & X[ju])).sum(axis=0), (w * (X[iu] ^ X[ju])).sum(axis=0)], axis=1)


def complement_adjacency(A: np.ndarray) -> np.ndarray:
    """Adjacency of the complement graph ("MIS on the dual graph")."""
    n = A.shape[0]
    return (1.0 - A) - np.eye(n)


def problem_adjacency(problem, A: np.ndarray) -> np.ndarray:
    """The adjacency the relaxed objective is built on (complement for max clique)."""
    return complement_adjacency(A) if _pid(problem) == MAXCLIQUE else A


# ------------------------------------------------------- energies (App. D)
def relaxed_objective(problem, A: np.ndarray, P: np.ndarray, lam: float = 2.0) -> np.ndarray:
    """l_hat(p) per replica. P is [N][S]; returns [S].

    MIS: -1^T p + lam * p^T A p / 2.
    Max-Cut: -sum_{i<j} A_ij (1 - (2p_i-1)(2p_j-1))/2, each undirected edge once.
    Max clique: MIS on the complement.
    """
    pid = _pid(problem)
    if pid in (MIS, MAXCLIQUE):
        B = problem_adjacency(pid, A)
        return -P.sum(axis=0) + lam * np.einsum("is,ij,js->s", P, B, P) / 2.0
    if pid == MAXCLIQUE_SPARSE:   # P:715 as printed: -1^T p + (lam/2)(1^T p (1^T p - 1) - p^T A p)
        T = P.sum(axis=0)
        return -T + lam / 2.0 * (T * (T - 1.0) - np.einsum("is,ij,js->s", P, A, P))
    if pid == MAXCUT:
        Z = 2.0 * P - 1.0
        iu, ju = np.nonzero(np.triu(A, 1))  # each undirected edge once (reading R15)
        w = A[iu, ju][:, None]
        return -(w * (1.0 - Z[iu] * Z[ju]) / 2.0).sum(axis=0)
    raise ValueError(problem)


def discrete_energy(problem, A: np.ndarray, X: np.ndarray, lam: float = 2.0) -> np.ndarray:
    """l(x) per replica at binary X [N][S] (Eq. 2 with the App. D energies)."""
    return relaxed_objective(problem, A, X.astype(np.float64), lam)


def printed_clique_energy(A: np.ndarray, x: np.ndarray, lam: float = 2.0) -> float:
    """The max-clique energy exactly as printed at P:715:
    -c^T x + (lam/2)(1^T x (1^T x - 1) - x^T A x)."""
    x = x.astype(np.float64)
    s = x.sum()
    return -s + lam / 2.0 * (s * (s - 1.0) - x @ A @ x)


def entropy(P: np.ndarray, alpha: int) -> np.ndarray:
    """alpha-entropy per replica (Eq. 7): sum_i 1 - (2 p_i - 1)^alpha."""
    return (1.0 - (2.0 * P - 1.0) ** alpha).sum(axis=0)


def std_rows(P: np.ndarray) -> np.ndarray:
    """Empirical population STD over replicas per variable, two-pass."""
    S = P.shape[1]
    mu = P.sum(axis=1) / S
    return np.sqrt(((P - mu[:, None]) ** 2).sum(axis=1) / S)


def comm_term(P: np.ndarray, comm: float) -> float:
    """-S * alpha_c * sum_i STD_i (Eq. 10)."""
    return -P.shape[1] * comm * std_rows(P).sum()


def R_hat(problem, A, P, gamma, alpha, lam, comm) -> float:
    """Ensemble objective (Eq. 10) = sum_s [l_hat_s + gamma s_s] + comm term."""
    return float((relaxed_objective(problem, A, P, lam) + gamma * entropy(P, alpha)).sum()
                 + comm_term(P, comm))


# ----------------------------------------------------- analytic gradients
def grad_objective(problem, A, P, lam) -> np.ndarray:
    """d l_hat / d p, [N][S].  MIS: -1 + lam (A p)_i ; Max-Cut: -deg_i + 2 (A p)_i."""
    pid = _pid(problem)
    if pid in (MIS, MAXCLIQUE):
        B = problem_adjacency(pid, A)
        return -1.0 + lam * (B @ P)
    if pid == MAXCLIQUE_SPARSE:   # d/dp_i of P:715 = -1 + (lam/2)(2 T - 1 - 2 (A p)_i), T = 1^T p per replica
        T = P.sum(axis=0)[None, :]
        return -1.0 + lam * ((T - 0.5) - A @ P)
    if pid == MAXCUT:
        return -A.sum(axis=1)[:, None] + 2.0 * (A @ P)
    raise ValueError(problem)


def grad_entropy(P, alpha) -> np.ndarray:
    """d s / d p = -2 alpha (2p - 1)^(alpha - 1)."""
    return -2.0 * alpha * (2.0 * P - 1.0) ** (alpha - 1)


def grad_comm(P, comm) -> np.ndarray:
    """d/dp_i^s of -S alpha_c STD_i = -alpha_c (p_i^s - mu_i) / STD_i (0 where STD_i < floor)."""
    S = P.shape[1]
    mu = P.sum(axis=1) / S
    sd = std_rows(P)
    out = np.zeros_like(P)
    ok = sd >= STD_FLOOR
    out[ok] = -comm * (P[ok] - mu[ok, None]) / sd[ok, None]
    return out


def grad_p(problem, A, P, gamma, alpha, lam, comm) -> np.ndarray:
    return grad_objective(problem, A, P, lam) + gamma * grad_entropy(P, alpha) + grad_comm(P, comm)


def sigmoid(theta):
    return 1.0 / (1.0 + np.exp(-theta))


def grad_theta(problem, A, theta, gamma, alpha, lam, comm) -> np.ndarray:
    """Chain rule through p = sigmoid(theta): dR/dtheta = dR/dp * p (1 - p)."""
    P = sigmoid(theta)
    return grad_p(problem, A, P, gamma, alpha, lam, comm) * P * (1.0 - P)


# -------------------------------------------------------------- optimizer
def adamw_step(theta, m, v, g, t, lr, beta1, beta2, eps, wd):
    """One AdamW step (Loshchilov & Hutter, cited at P:221), t = 1, 2, ...

    theta <- theta (1 - lr wd);  m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;
    theta <- theta - lr * mhat / (sqrt(vhat) + eps),  mhat = m/(1-b1^t), vhat = v/(1-b2^t).
    """
    theta = theta * (1.0 - lr * wd)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** t)
    vhat = v / (1.0 - beta2 ** t)
    theta = theta - lr * mhat / (np.sqrt(vhat) + eps)
    return theta, m, v


def gamma_schedule(gamma_min: float, gamma_max: float, total: int) -> np.ndarray:
    """Linear gamma, both endpoints used (reading R10)."""
    if total == 1:
        return np.array([gamma_min], dtype=np.float64)
    return gamma_min + (gamma_max - gamma_min) * np.arange(total) / (total - 1)


# ----------------------------------------------------------- initial state
def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def init_theta(n: int, S_total: int, seed: int, lo: float = -0.01, hi: float = 0.01) -> np.ndarray:
    """theta_0[i][s] ~ U(lo, hi) from a counter hash (BASELINE.json configs[0]; paper silent).

    key = splitmix64(seed) + i*S_total + s;  k = top 24 bits of splitmix64(key);
    theta = lo + (hi - lo) * k * 2^-24.  Returned in fp64 (exact values of the
    fp32 contract's double intermediate before its final rounding)."""
    base = _splitmix64(np.array([seed], dtype=np.uint64))[0]
    i = np.arange(n, dtype=np.uint64)[:, None]
    s = np.arange(S_total, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = base + i * np.uint64(S_total) + s
    k = (_splitmix64(key) >> np.uint64(40)).astype(np.float64)
    lo64, hi64 = float(np.float32(lo)), float(np.float32(hi))
    return lo64 + (hi64 - lo64) * k * 2.0 ** -24


def init_p_clamp(n: int, S_total: int, seed: int, lo: float = -0.01, hi: float = 0.01) -> np.ndarray:
    """Clamp map (NEXT-1): the parameter is p itself, p_0 = 1/2 + U(lo, hi) from the same
    counter hash as init_theta (reading R23: the paper's init for Clamp is not printed)."""
    return 0.5 + init_theta(n, S_total, seed, lo, hi)


def clamp01(w):
    """Clamp(w) into [0, 1]."""
    return np.clip(w, 0.0, 1.0)


# ------------------------------------------------------------ Langevin noise
NOISE_SALT = 0x6A09E667F3BCC909


def _box_muller_pair(h: np.ndarray):
    """Both Box-Muller outputs of one hash: u1 = (h >> 40 + 1) 2^-24 in (0, 1], u2 = ((h >> 16) & (2^24 - 1))
    2^-24 in [0, 1); r = sqrt(-2 ln u1); (r cos 2 pi u2, r sin 2 pi u2) -- two independent N(0, 1)."""
    u1 = ((h >> np.uint64(40)) + np.uint64(1)).astype(np.float64) * 2.0 ** -24
    u2 = ((h >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float64) * 2.0 ** -24
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2)


def gauss_noise(seed: int, t: int, n: int, S_total: int) -> np.ndarray:
    """xi ~ N(0, 1) [n][S_total] for Adam step t by Box-Muller in fp64 from a counter hash. Replicas pair up
    (s even, s + 1) on one hash h = splitmix64(splitmix64(seed ^ salt) + (t n + i) S_total + s_even):
    xi = r cos 2 pi u2 for the even replica and r sin 2 pi u2 for the odd one (reading R24)."""
    base = _splitmix64(np.array([(seed ^ NOISE_SALT) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    i = np.arange(n, dtype=np.uint64)[:, None]
    s = np.arange(S_total, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        key = base + (np.uint64(t) * np.uint64(n) + i) * np.uint64(S_total) + (s & ~np.uint64(1))
    zc, zs = _box_muller_pair(_splitmix64(key))
    return np.where((s & np.uint64(1)) == 0, zc, zs)


# --------------------------------------------------------------- the loop
def run(problem, A, theta0, gammas, alpha=2, lam=2.0, comm=0.1, lr=1.0, beta1=0.9,
        beta2=0.999, eps=1e-8, wd=0.01, m0=None, v0=None, t0=0, map="sigmoid", temperature=0.0, seed=0):
    """PQQA with AdamW, fp64. Returns (theta, m, v).

    map="sigmoid": theta is the parameter, p = sigmoid(theta), gradient by the chain rule.
    map="clamp" (sensitive transition, Eq. 11): ``theta0`` is p_0; AdamW is applied to p with
    dR/dp, then p <- Clamp(p'); the returned "theta" is p.
    temperature > 0: + sqrt(2 lr T) xi after the optimizer step, before the map (Eq. 9 / 11)."""
    theta = np.array(theta0, dtype=np.float64)
    m = np.zeros_like(theta) if m0 is None else np.array(m0, dtype=np.float64)
    v = np.zeros_like(theta) if v0 is None else np.array(v0, dtype=np.float64)
    n, S = theta.shape
    for k, gamma in enumerate(gammas):
        t = t0 + k + 1
        if map == "clamp":
            g = grad_p(problem, A, theta, float(gamma), alpha, lam, comm)
        else:
            g = grad_theta(problem, A, theta, float(gamma), alpha, lam, comm)
        theta, m, v = adamw_step(theta, m, v, g, t, lr, beta1, beta2, eps, wd)
        if temperature > 0.0:
            theta = theta + np.sqrt(2.0 * lr * temperature) * gauss_noise(seed, t, n, S)
        if map == "clamp":
            theta = clamp01(theta)
    return theta, m, v


def round_x(theta: np.ndarray, map="sigmoid") -> np.ndarray:
    """x = Theta(p - 1/2) with Theta(0)=1 (reading R12): theta >= 0 for the sigmoid
    map, p >= 1/2 for clamp (theta holds p)."""
    return (theta >= (0.5 if map == "clamp" else 0.0)).astype(np.int64)


def counts(problem, A: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Per replica [S][3] = (size, violations, cut), each undirected edge once.

    violations: #{(i<j) in E' : x_i = x_j = 1} with E' = E (MIS, Max-Cut) or the
    complement (max clique); cut: #{(i<j) in E : x_i != x_j}."""
    pid = _pid(problem)
    if pid == MAXCLIQUE_SPARSE:   # the same counts as max clique on the complement
        return counts(MAXCLIQUE, A, X)
    B = problem_adjacency(pid, A)
    X = X.astype(np.int64)
    n, S = X.shape
    out = np.zeros((S, 3), dtype=np.int64)
    iu, ju = np.nonzero(np.triu(B, 1))
    for s in range(S):
        x = X[:, s]
        out[s, 0] = x.sum()
        out[s, 1] = int((x[iu] & x[ju]).sum())
        if pid == MAXCUT:
            ia, ja = np.nonzero(np.triu(A, 1))
            out[s, 2] = int((x[ia] ^ x[ja]).sum())
        else:
            out[s, 2] = int((x[iu] ^ x[ju]).sum())
    return out


def energy_from_counts(problem, c: np.ndarray, lam: float = 2.0) -> np.ndarray:
    pid = _pid(problem)
    if pid == MAXCUT:
        return -c[:, 2].astype(np.float64)
    return -c[:, 0].astype(np.float64) + lam * c[:, 1].astype(np.float64)


def best_replica(energies: np.ndarray) -> int:
    """argmin energy, lowest replica index on ties (reading R13)."""
    return int(np.flatnonzero(energies == energies.min())[0])


def brute_force(problem, A: np.ndarray, lam: float = 2.0):
    """Exhaustive argmin of the discrete energy l(x) over {0,1}^N (N <= 20).

    Returns (min_energy, list of minimisers)."""
    n = A.shape[0]
    if n > 22:
        raise ValueError("brute force limited to N <= 22")
    best, arg = np.inf, []
    X = np.array(list(itertools.product([0, 1], repeat=n)), dtype=np.float64).T  # [N][2^N]
    E = relaxed_objective(problem, A, X, lam)
    best = E.min()
    arg = [X[:, k].astype(np.int64) for k in np.flatnonzero(np.isclose(E, best, atol=1e-9))]
    return float(best), arg


# ======================================================= K-ary (NEXT-4)
# Generalisation to discrete variables x_i in {0..K-1} (Appendix B): each
# variable is relaxed to a row of K probabilities P[i, s, :] (one-hot encoding), the
# entropy becomes s_K (Eq. after), the map is Clamp-then-normalise,
# and the sensitive transition (Eq. 11) applies AdamW to P itself. Graph colouring
# (P:745-750): conflicts = #{(i<j) in E : x_i = x_j}, relaxed as
# sum_{(i<j) in E} sum_k p_ik p_jk (exact at one-hot P). Arrays are [N][S][K].
def c_K(K: int, alpha: int) -> float:
    """Normaliser of s_K: 1 / ((K-1) ((K-1)^(alpha-1) + 1))."""
    return 1.0 / ((K - 1) * ((K - 1) ** (alpha - 1) + 1))


def entropy_K(P: np.ndarray, alpha: int) -> np.ndarray:
    """s_K per replica: sum_i 1 - c_K sum_k (K p_ik - 1)^alpha."""
    K = P.shape[2]
    return (1.0 - c_K(K, alpha) * ((K * P - 1.0) ** alpha).sum(axis=2)).sum(axis=0)


def coloring_objective(A: np.ndarray, P: np.ndarray) -> np.ndarray:
    """Relaxed conflicts per replica: sum_{(i<j) in E} sum_k p_ik p_jk = (1/2) sum_ij A_ij <p_i, p_j>."""
    return 0.5 * np.einsum("isk,ij,jsk->s", P, A, P)


def std_rows_K(P: np.ndarray) -> np.ndarray:
    """Population STD over replicas of every (i, k) (Eq. 10 applied per colour column)."""
    S = P.shape[1]
    mu = P.sum(axis=1) / S
    return np.sqrt(((P - mu[:, None, :]) ** 2).sum(axis=1) / S)


def R_hat_K(A, P, gamma, alpha, comm) -> float:
    """sum_s [l(P_s) + gamma s_K(P_s)] - S alpha_c sum_{i,k} STD_ik."""
    return float((coloring_objective(A, P) + gamma * entropy_K(P, alpha)).sum()
                 - P.shape[1] * comm * std_rows_K(P).sum())


def grad_K(A, P, gamma, alpha, comm) -> np.ndarray:
    """dR/dP [N][S][K]: (A P)_isk - gamma c_K alpha K (K p - 1)^(alpha-1) - alpha_c (p - mu_ik)/STD_ik."""
    K, S = P.shape[2], P.shape[1]
    obj = np.einsum("ij,jsk->isk", A, P)
    ent = -c_K(K, alpha) * alpha * K * (K * P - 1.0) ** (alpha - 1)
    mu = P.sum(axis=1) / S
    sd = std_rows_K(P)
    com = np.zeros_like(P)
    ok = sd >= STD_FLOOR
    d = P - mu[:, None, :]
    com[:, :, :] = np.where(ok[:, None, :], -comm * d / np.where(ok, sd, 1.0)[:, None, :], 0.0)
    return obj + gamma * ent + com


def grad_K_map(A, P, gamma, alpha, comm) -> np.ndarray:
    """The K-ary gradient through the map (reading R33): with W = P on the simplex (the sensitive
    transition replaces W by sigma(W) every step), d sigma_k' / d W_k = delta_kk' - P_k' inside the clamp
    range, so dR/dW = g - <g, P> per (variable, replica) row, g = dR/dP (grad_K)."""
    g = grad_K(A, P, gamma, alpha, comm)
    return g - (g * P).sum(axis=2, keepdims=True)


def clamp_normalize(W: np.ndarray) -> np.ndarray:
    """sigma(W_ik) = Clamp(W_ik) / sum_k' Clamp(W_ik'); a row whose clamps are all 0 maps
    to the uniform 1/K (reading R27: the paper leaves 0/0 undefined)."""
    K = W.shape[-1]
    C = np.clip(W, 0.0, 1.0)
    Z = C.sum(axis=-1, keepdims=True)
    return np.where(Z > 0, C / np.where(Z > 0, Z, 1.0), 1.0 / K)


def init_W_K(n: int, S_total: int, K: int, seed: int, lo: float = -0.01, hi: float = 0.01) -> np.ndarray:
    """W_0[i][s][k] = 1/K + U(lo, hi), U from the counter hash keyed (seed, i K + k, s):
    key = splitmix64(seed) + (i K + k) S_total + s; k24 = top 24 bits; u = lo + (hi - lo) k24 2^-24."""
    base = _splitmix64(np.array([seed], dtype=np.uint64))[0]
    i = np.arange(n, dtype=np.uint64)[:, None, None]
    s = np.arange(S_total, dtype=np.uint64)[None, :, None]
    k = np.arange(K, dtype=np.uint64)[None, None, :]
    with np.errstate(over="ignore"):
        key = base + (i * np.uint64(K) + k) * np.uint64(S_total) + s
    k24 = (_splitmix64(key) >> np.uint64(40)).astype(np.float64)
    lo64, hi64 = float(np.float32(lo)), float(np.float32(hi))
    return 1.0 / K + (lo64 + (hi64 - lo64) * k24 * 2.0 ** -24)


def gauss_noise_K(seed: int, t: int, n: int, S_total: int, K: int) -> np.ndarray:
    """xi [n][S][K] of the K-ary path: colours pair up (k even, k + 1) on one hash
    h = splitmix64(splitmix64(seed ^ salt) + ((t n + i) K + k_even) S_total + s); cos for even k, sin for odd."""
    base = _splitmix64(np.array([(seed ^ NOISE_SALT) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    i = np.arange(n, dtype=np.uint64)[:, None, None]
    s = np.arange(S_total, dtype=np.uint64)[None, :, None]
    k = np.arange(K, dtype=np.uint64)[None, None, :]
    with np.errstate(over="ignore"):
        key = base + ((np.uint64(t) * np.uint64(n) + i) * np.uint64(K) + (k & ~np.uint64(1))) * np.uint64(S_total) + s
    zc, zs = _box_muller_pair(_splitmix64(key))
    return np.where((k & np.uint64(1)) == 0, zc, zs)


def run_K(A, P0, gammas, alpha=2, comm=0.1, lr=1.0, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.01,
          m0=None, v0=None, t0=0, temperature=0.0, seed=0, through_map=True):
    """K-ary PQQA, fp64: AdamW on the parameter W = P with the gradient through the map (grad_K_map,
    reading R33; through_map=False: dR/dP itself, reading R29), (+ noise), then P <- clamp_normalize(P')
    (the sensitive transition with the K-ary map of P:672-676). P0 is the (already normalised) starting
    point. Returns (P, m, v)."""
    P = np.array(P0, dtype=np.float64)
    m = np.zeros_like(P) if m0 is None else np.array(m0, dtype=np.float64)
    v = np.zeros_like(P) if v0 is None else np.array(v0, dtype=np.float64)
    n, S, K = P.shape
    for k, gamma in enumerate(gammas):
        t = t0 + k + 1
        g = (grad_K_map if through_map else grad_K)(A, P, float(gamma), alpha, comm)
        P, m, v = adamw_step(P, m, v, g, t, lr, beta1, beta2, eps, wd)
        if temperature > 0.0:
            P = P + np.sqrt(2.0 * lr * temperature) * gauss_noise_K(seed, t, n, S, K)
        P = clamp_normalize(P)
    return P, m, v


def round_K(P: np.ndarray) -> np.ndarray:
    """x_is = argmax_k p_isk, lowest k on ties."""
    return np.argmax(P, axis=2).astype(np.int64)


def conflicts(A: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Per replica: #{(i<j) in E : x_i = x_j} (the colouring cost, read as minimised)."""
    iu, ju = np.nonzero(np.triu(A, 1))
    return (X[iu] == X[ju]).sum(axis=0).astype(np.int64)


def brute_force_coloring(A: np.ndarray, K: int) -> int:
    """Minimum conflicts over all K^N colourings (K^N <= 2e6)."""
    n = A.shape[0]
    if K ** n > 2_000_000:
        raise ValueError("brute force too large")
    iu, ju = np.nonzero(np.triu(A, 1))
    X = np.array(list(itertools.product(range(K), repeat=n)), dtype=np.int64).T  # [N][K^N]
    return int((X[iu] == X[ju]).sum(axis=0).min())
