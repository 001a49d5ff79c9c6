"""numpy/scipy restatement of the reference hot path (test infrastructure only).

Every function mirrors one reference function operation for operation (the
cited file:line is relative to ``/root/reference/pkg/src/cscluster/``), so
results are bit-identical to the reference on the same library build.  Graphs
are plain ``Csr`` tuples; nothing here touches the GPU or the product package.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

TINY = np.finfo(np.float64).tiny


# ---------------------------------------------------------------------------
# graph (graph.py)


@dataclass
class Csr:
    num_nodes: int
    indptr: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    degrees: np.ndarray

    @property
    def matrix(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.weights, self.indices, self.indptr), shape=(self.num_nodes, self.num_nodes))

    @property
    def dis(self) -> np.ndarray:
        """d^-1/2 with 0 on isolated nodes (graph.py:166-168)."""
        d = self.degrees
        with np.errstate(divide="ignore"):
            return np.where(d > 0, 1.0 / np.sqrt(np.where(d > 0, d, 1.0)), 0.0)


def csr_from_scipy(A, num_nodes: int) -> Csr:
    """graph.py:58-70."""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    A.eliminate_zeros()
    deg = np.asarray(A.sum(axis=1)).ravel().astype(np.float64)
    return Csr(num_nodes, A.indptr.copy(), A.indices.copy(), A.data.astype(np.float64, copy=True), deg)


def build_csr(src, dst, w, num_nodes: int) -> Csr:
    """Canonical CSR of validated, loop-free edge triples (graph.py:122-125)."""
    A = sp.coo_matrix((w, (src, dst)), shape=(num_nodes, num_nodes)).tocsr()
    A.sum_duplicates()
    return csr_from_scipy(A.maximum(A.T), num_nodes)


def sbm_csr(src, dst, num_nodes: int) -> Csr:
    """SBM path: each pair generated once, W = A + A^T (sbm.py:147-155)."""
    A = sp.coo_matrix((np.ones(src.size), (src, dst)), shape=(num_nodes, num_nodes)).tocsr()
    return csr_from_scipy(A + A.T, num_nodes)


def csr_digest(g: Csr) -> str:
    h = hashlib.sha256()
    for a in (np.asarray(g.indptr, np.int64), np.asarray(g.indices, np.int64), g.weights, g.degrees):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


class EdgeListError(ValueError):
    """The reference's GraphError for edge-list lines (graph.py:203, 209)."""


def parse_edge_text(text: str, name: str = "<path>"):
    """read_edge_list's line loop (graph.py:188-212) over already-decoded text: (rows E x 3
    float64, header node count or None).  ``text.splitlines(keepends=True)`` restricted to
    '\n', '\r\n' and '\r' is Python's universal-newline iteration of the file object."""
    import io

    rows = []
    header_nodes = None
    for lineno, line in enumerate(io.StringIO(text, newline=None), start=1):
        stripped = line.strip()
        if not stripped:
            continue
        if stripped.startswith("#"):
            parts = stripped[1:].split()
            if len(parts) == 2 and parts[0] == "nodes":
                try:
                    header_nodes = int(parts[1])
                except ValueError:
                    pass
            continue
        parts = stripped.split()
        if len(parts) not in (2, 3):
            raise EdgeListError(f"{name}:{lineno}: expected 'src dst [weight]', got {stripped!r}")
        try:
            i = int(parts[0])
            j = int(parts[1])
            w = float(parts[2]) if len(parts) == 3 else 1.0
        except ValueError as exc:
            raise EdgeListError(f"{name}:{lineno}: {exc}") from None
        rows.append((i, j, w))
    return np.array(rows, dtype=np.float64).reshape(len(rows), 3), header_nodes


def format_edge_list(num_nodes: int, indptr, indices, weights) -> bytes:
    """write_edge_list's bytes (graph.py:215-225): W.tocoo() of a canonical CSR is its storage
    order, so entries with row < col in CSR order, one "i j repr(w)" line each."""
    out = [f"# nodes {num_nodes}\n"]
    for i in range(num_nodes):
        for k in range(int(indptr[i]), int(indptr[i + 1])):
            j = int(indices[k])
            if i < j:
                out.append(f"{i} {j} {float(weights[k])!r}\n")
    return "".join(out).encode("utf-8")


def laplacian_apply(g: Csr, x: np.ndarray, W=None, dis=None) -> np.ndarray:
    """x - dis * (W @ (dis * x))  (graph.py:147-155)."""
    x = np.asarray(x, dtype=np.float64)
    W = g.matrix if W is None else W
    dis = g.dis if dis is None else dis
    if x.ndim == 1:
        return x - dis * (W @ (dis * x))
    return x - dis[:, None] * (W @ (dis[:, None] * x))


def dense_laplacian(g: Csr) -> np.ndarray:
    """Loop-built dense L (reference tests/helpers.py:22-35 style)."""
    n = g.num_nodes
    W = np.zeros((n, n))
    for i in range(n):
        for e in range(g.indptr[i], g.indptr[i + 1]):
            W[i, g.indices[e]] = g.weights[e]
    d = W.sum(axis=1)
    L = np.eye(n)
    nz = np.nonzero(W)
    for i, j in zip(*nz):
        if d[i] > 0 and d[j] > 0:
            L[i, j] -= W[i, j] / np.sqrt(d[i] * d[j])
    return L


# ---------------------------------------------------------------------------
# filters (filters.py)


def jackson(order: int) -> np.ndarray:
    """filters.py:94-99."""
    q = order + 2
    l = np.arange(order + 1)
    ang = np.pi * l / q
    return ((q - l) * np.cos(ang) + np.sin(ang) / np.tan(np.pi / q)) / q


def lowpass_coeffs(cutoff: float, order: int, damping: str = "jackson") -> np.ndarray:
    """filters.py:102-117."""
    theta_c = np.arccos(cutoff - 1.0)
    l = np.arange(1, order + 1)
    c = np.empty(order + 1)
    c[0] = 1.0 - theta_c / np.pi
    c[1:] = -2.0 * np.sin(l * theta_c) / (np.pi * l)
    if damping == "jackson":
        c = c * jackson(order)
    return c


def highpass_coeffs(low: np.ndarray) -> np.ndarray:
    """filters.py:125-137."""
    c = -low.copy()
    c[0] += 1.0
    return c


def evaluate(coeffs: np.ndarray, lam) -> np.ndarray:
    """filters.py:43-57."""
    y = np.asarray(lam, dtype=np.float64) - 1.0
    out = np.full_like(y, coeffs[0])
    if coeffs.size > 1:
        t_prev = np.ones_like(y)
        t_cur = y.copy()
        out = out + coeffs[1] * t_cur
        for l in range(2, coeffs.size):
            t_prev, t_cur = t_cur, 2.0 * y * t_cur - t_prev
            out = out + coeffs[l] * t_cur
    return out


def psd_ridge(coeffs: np.ndarray, grid_points: int = 2001) -> float:
    """filters.py:248-256."""
    lo = float(np.min(evaluate(coeffs, np.linspace(0.0, 2.0, grid_points))))
    return max(0.0, -lo) + 1e-8


def apply_filter(coeffs: np.ndarray, g: Csr, x: np.ndarray, W=None, dis=None) -> np.ndarray:
    """Chebyshev recurrence with y = L - I (filters.py:140-155)."""
    x = np.asarray(x, dtype=np.float64)
    W = g.matrix if W is None else W
    dis = g.dis if dis is None else dis
    c = coeffs
    out = c[0] * x
    if c.size > 1:
        t_prev = x
        t_cur = laplacian_apply(g, x, W, dis) - x
        out = out + c[1] * t_cur
        for l in range(2, c.size):
            t_prev, t_cur = t_cur, 2.0 * (laplacian_apply(g, t_cur, W, dis) - t_cur) - t_prev
            out = out + c[l] * t_cur
    return out


def apply_filter_threaded(coeffs: np.ndarray, g: Csr, x: np.ndarray, threads: int) -> np.ndarray:
    """apply_filter on column slices in parallel threads (the filter is columnwise,
    filters.py:140; scipy's CSR @ dense releases the GIL).  Used only as the timed
    CPU reference arm, so the reference algorithm gets every host core."""
    from concurrent.futures import ThreadPoolExecutor

    W, dis = g.matrix, g.dis
    cols = np.array_split(np.arange(x.shape[1]), max(1, min(threads, x.shape[1])))
    parts = [np.ascontiguousarray(x[:, c]) for c in cols]
    with ThreadPoolExecutor(len(parts)) as ex:
        outs = list(ex.map(lambda p: apply_filter(coeffs, g, p, W, dis), parts))
    return np.concatenate(outs, axis=1)


# ---------------------------------------------------------------------------
# spectrum (spectrum.py)


def round_half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


def default_probe_signals(n: int) -> int:
    """spectrum.py:53-55."""
    return 2 * int(math.ceil(math.log(max(n, 2))))


def eigencount(g: Csr, lam: float, order: int, ds: int, rng: np.random.Generator, W=None, dis=None) -> float:
    """spectrum.py:58-87 (count before rounding)."""
    c = lowpass_coeffs(min(lam, 2.0 - 1e-12), order, "jackson")
    signals = rng.standard_normal((g.num_nodes, ds)) / np.sqrt(ds)
    filtered = apply_filter(c, g, signals, W, dis)
    return float(np.sum(filtered * filtered))


def estimate_lambda_k(g: Csr, k: int, order: int, ds: int | None, rng, max_steps: int = 20, refine: bool = False):
    """spectrum.py:90-140 -> (lambda_hat, trace, warning)."""
    ds = ds if ds is not None else default_probe_signals(g.num_nodes)
    W, dis = g.matrix, g.dis
    lo, hi = 0.0, 2.0
    trace: list[tuple[float, float]] = []

    def probe(lam):
        cnt = eigencount(g, lam, order, ds, rng, W, dis)
        trace.append((float(lam), cnt))
        return cnt

    for _ in range(max_steps):
        mid = 0.5 * (lo + hi)
        r = round_half_up(probe(mid))
        if r == k:
            lam_hat = mid
            if refine and (hi - lo) > 0.01:
                mid2 = 0.5 * (lo + mid)
                if round_half_up(probe(mid2)) == k:
                    lam_hat = mid2
            return lam_hat, trace, False
        if r > k:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi), trace, True


# ---------------------------------------------------------------------------
# features (features.py)


def gaussian_signals(n: int, d: int, seed) -> np.ndarray:
    """features.py:61-63."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, d)) / np.sqrt(d)


def build_features(coeffs: np.ndarray, g: Csr, signals: np.ndarray):
    """features.py:70-93 -> (rows, zero_rows)."""
    filtered = apply_filter(coeffs, g, signals)
    norms = np.linalg.norm(filtered, axis=1)
    zero_rows = np.flatnonzero(norms <= 1e-300)
    safe = norms.copy()
    safe[zero_rows] = 1.0
    rows = filtered / safe[:, None]
    rows[zero_rows] = 0.0
    return rows, zero_rows


# ---------------------------------------------------------------------------
# sampling (sampling.py)


def draw_sampling(num_nodes: int, n: int, seed, exclude=None) -> np.ndarray:
    """sampling.py:64-88."""
    rng = np.random.default_rng(seed)
    if exclude is not None and len(exclude):
        eligible = np.setdiff1d(np.arange(num_nodes), np.asarray(exclude, dtype=np.int64))
        idx = eligible[rng.choice(eligible.size, size=n, replace=False)]
    else:
        idx = rng.choice(num_nodes, size=n, replace=False)
    return idx.astype(np.int64)


def system_apply(g: Csr, hp: np.ndarray, gamma: float, ridge: float, mask: np.ndarray, X: np.ndarray, W=None,
                 dis=None) -> np.ndarray:
    """sampling.py:119-121."""
    reg = apply_filter(hp, g, X, W, dis) + ridge * X
    return mask[:, None] * X + gamma * reg


def interpolate_all(g: Csr, hp: np.ndarray, gamma: float, ridge: float, indices: np.ndarray, reduced: np.ndarray,
                    tol: float = 1e-6, max_iters: int = 1000):
    """sampling.py:124-180 -> (X, iterations, residuals, converged)."""
    n, k = reduced.shape
    N = g.num_nodes
    W, dis = g.matrix, g.dis
    mask = np.zeros(N)
    mask[indices] = 1.0
    B = np.zeros((N, k))
    B[indices] = reduced
    X = np.zeros((N, k))
    R = B.copy()
    P = R.copy()
    rs = np.einsum("ij,ij->j", R, R)
    target2 = (tol * np.sqrt(np.einsum("ij,ij->j", B, B))) ** 2
    conv_at = np.zeros(k, dtype=np.int64)
    active = rs > target2
    iters = 0
    while active.any() and iters < max_iters:
        AP = system_apply(g, hp, gamma, ridge, mask, P, W, dis)
        denom = np.einsum("ij,ij->j", P, AP)
        alpha = np.where(active & (np.abs(denom) > TINY), rs / np.where(np.abs(denom) > TINY, denom, 1.0), 0.0)
        X += alpha * P
        R -= alpha * AP
        rs_new = np.einsum("ij,ij->j", R, R)
        beta = np.where(active, rs_new / np.maximum(rs, TINY), 0.0)
        P = R + beta * P
        rs = rs_new
        iters += 1
        done = active & (rs <= target2)
        conv_at[done] = iters
        active = active & ~done
    residuals = np.sqrt(rs)
    converged = residuals <= np.sqrt(target2) + TINY
    conv_at[active] = iters
    return X, conv_at, residuals, converged


def assign(soft: np.ndarray):
    """sampling.py:197-220 -> (labels, fallback)."""
    soft = np.asarray(soft, dtype=np.float64)
    norms = np.linalg.norm(soft, axis=0)
    if not np.any(norms > 0):
        raise ValueError("all indicator vectors are zero")
    normalized = soft / np.where(norms > 0, norms, 1.0)[None, :]
    normalized[:, norms == 0] = -np.inf
    labels = normalized.argmax(axis=1)
    fallback = np.flatnonzero(np.all(soft == 0.0, axis=1))
    if fallback.size:
        labels[fallback] = soft[fallback].argmax(axis=1)
    return labels, fallback


# ---------------------------------------------------------------------------
# k-means (kmeans.py)


def _sq_dists(points, centroids):
    """kmeans.py:39-43."""
    pp = (points * points).sum(axis=1)[:, None]
    cc = (centroids * centroids).sum(axis=1)[None, :]
    return np.maximum(pp + cc - 2.0 * points @ centroids.T, 0.0)


def _seed_kmeanspp(points, k, rng):
    """kmeans.py:46-61 (k-means++ branch)."""
    q = points.shape[0]
    cent = np.empty((k, points.shape[1]))
    cent[0] = points[rng.integers(q)]
    d2 = ((points - cent[0]) ** 2).sum(axis=1)
    for j in range(1, k):
        total = d2.sum()
        cent[j] = points[rng.choice(q, p=d2 / total)] if total > 0 else points[rng.integers(q)]
        d2 = np.minimum(d2, ((points - cent[j]) ** 2).sum(axis=1))
    return cent


def _lloyd(points, cent, max_iters, tol):
    """kmeans.py:64-93."""
    q, k = points.shape[0], cent.shape[0]
    labels = np.zeros(q, dtype=np.int64)
    inertia = np.inf
    iters = 0
    for it in range(max_iters):
        D = _sq_dists(points, cent)
        labels = D.argmin(axis=1)
        pd2 = D[np.arange(q), labels]
        new = float(pd2.sum())
        iters = it + 1
        repaired = False
        counts = np.bincount(labels, minlength=k)
        for j in range(k):
            if counts[j] > 0:
                cent[j] = points[labels == j].mean(axis=0)
            else:
                far = int(pd2.argmax())
                cent[j] = points[far]
                pd2[far] = 0.0
                repaired = True
        if not repaired and inertia - new <= tol * max(new, np.finfo(float).tiny):
            inertia = new
            break
        inertia = new
    return labels, inertia, iters


def kmeans(points, k: int, seed: int, replicates: int = 20, max_iters: int = 100, tol: float = 1e-6):
    """kmeans.py:96-126 (k-means++ seeding) -> (labels, inertia, iterations)."""
    points = np.asarray(points, dtype=np.float64)
    best = None
    for ss in np.random.SeedSequence(seed).spawn(replicates):
        rng = np.random.default_rng(ss)
        lab, inert, its = _lloyd(points, _seed_kmeanspp(points, k, rng), max_iters, tol)
        if best is None or inert < best[1]:
            best = (lab, inert, its)
    return best


# ---------------------------------------------------------------------------
# rng + pipeline (_rng.py, pipeline.py)


def substream_seq(seed: int, stage: str) -> np.random.SeedSequence:
    """_rng.py:10-21."""
    dig = hashlib.sha256(stage.encode("utf-8")).digest()
    words = tuple(int.from_bytes(dig[i : i + 4], "little") for i in range(0, 16, 4))
    return np.random.SeedSequence((int(seed),) + words)


def substream(seed: int, stage: str) -> np.random.Generator:
    return np.random.default_rng(substream_seq(seed, stage))


def substream_seed(seed: int, stage: str) -> int:
    """_rng.py:24-28."""
    state = substream_seq(seed, stage).generate_state(2, dtype=np.uint64)
    return int(state[0] ^ (state[1] >> 1))


def run_csc(g: Csr, k: int, d: int | None = None, n: int | None = None, p: int = 50, gamma: float = 1e-3,
            seed: int = 0, lambda_k: float | None = None, tol: float = 1e-6, max_iters: int = 1000) -> dict:
    """pipeline.py:113-225 (gaussian signals, Jackson damping, default k-means)."""
    N = g.num_nodes
    n = n if n is not None else min(int(math.ceil(2.0 * k * math.log(k))), N)
    d = d if d is not None else int(math.ceil(4.0 * math.log(max(n, 2))))
    if lambda_k is None:
        lam, trace, warn = estimate_lambda_k(g, k, p, None, substream(seed, "probe"))
    else:
        lam, trace, warn = float(lambda_k), [], False
    low = lowpass_coeffs(lam, p, "jackson")
    high = highpass_coeffs(low)
    signals = gaussian_signals(N, d, substream(seed, "signals"))
    rows, zero_rows = build_features(low, g, signals)
    idx = draw_sampling(N, n, substream(seed, "sampling"), exclude=zero_rows)
    km_labels, inertia, km_iters = kmeans(rows[idx], k, substream_seed(seed, "kmeans"))
    reduced = np.zeros((n, k))
    reduced[np.arange(n), km_labels] = 1.0
    ridge = psd_ridge(high)
    X, its, res, conv = interpolate_all(g, high, gamma, ridge, idx, reduced, tol, max_iters)
    labels, fallback = assign(X)
    return {
        "lambda_k_hat": lam, "trace": trace, "lambda_warning": warn, "features": rows, "zero_rows": zero_rows,
        "indices": idx, "kmeans_labels": km_labels, "kmeans_inertia": inertia, "kmeans_iterations": km_iters,
        "ridge": ridge, "soft": X, "solver_iterations": its, "solver_residuals": res, "solver_converged": conv,
        "labels": labels, "fallback": fallback, "d": d, "n": n,
    }
