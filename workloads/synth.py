"""Counter-based synthetic workloads (SURVEY.md §8(d) "Synthetic inputs" / "Two generators" / "Configs").

Every row is a pure function of (model_seed, row_seed, row index): rows are drawn in fixed blocks of
BLOCK rows, each block from its own Philox stream keyed by (row_seed, block), so any slice can be
regenerated on any host without generating the rows before it.

G-LM (latent-manifold mixture, the default "realistic" generator):
    latent  z = mu_c + 0.6 * eps,        mu_c ~ N(0, I_l),  c ~ U{0..n_comp-1}, eps ~ N(0, I_l)
    vector  x = s * (z @ W) + m + sigma * eta,   W_ij ~ N(0, 1/l),  eta ~ N(0, I_D)
    variants: integer (round + clip to [0,255], SIFT-like), normalize (L2-normalise, Deep-like),
              OOD queries (mu'_c = mu_c + delta, delta ~ N(0, 0.5^2 I_l), Text2Image-like).
G-CL (clustered low-rank, the stress generator):
    x = center_c + 40 * (u @ B_c) + N(0, 4^2),  center_c ~ N(64, 25^2)^D, B_c a random orthonormal
    rank-12 basis per cluster, u ~ N(0, I_12).

Nothing here computes a distance, a neighbour, or any step of the method.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

BLOCK = 1 << 18          # rows per Philox stream
_MODEL_STREAM = 0x4D4F44454C  # "MODEL"
_ROW_STREAM = 0x524F5753      # "ROWS"


def _rng(seed: int, stream: int, sub: int = 0) -> np.random.Generator:
    key = np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF),
                    np.uint64(((stream & 0xFFFFFFFF) << 32) | (sub & 0xFFFFFFFF))], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


@dataclasses.dataclass(frozen=True)
class GLM:
    dim: int
    ell: int = 32
    s: float = 30.0
    m: float = 64.0
    sigma: float = 2.0
    n_comp: int = 1000
    integer: bool = False
    normalize: bool = False

    def _model(self, model_seed: int):
        g = _rng(model_seed, _MODEL_STREAM, 0)
        mu = g.standard_normal((self.n_comp, self.ell))
        w = g.standard_normal((self.ell, self.dim)) / np.sqrt(self.ell)
        delta = 0.5 * g.standard_normal(self.ell)
        return mu, w, delta

    def rows(self, model_seed: int, row_seed: int, start: int, n: int, ood: bool = False) -> np.ndarray:
        mu, w, delta = self._model(model_seed)
        if ood:
            mu = mu + delta[None, :]
        w32 = w.astype(np.float32)
        out = np.empty((n, self.dim), dtype=np.float32)
        b0, b1 = start // BLOCK, (start + n - 1) // BLOCK if n > 0 else start // BLOCK - 1

        def block(b):  # rows of Philox block b that fall in [start, start + n): independent of every other block
            g = _rng(row_seed, _ROW_STREAM, b)
            comp = g.integers(0, self.n_comp, size=BLOCK)
            eps = g.standard_normal((BLOCK, self.ell), dtype=np.float32)
            eta = g.standard_normal((BLOCK, self.dim), dtype=np.float32)
            lo = max(start, b * BLOCK) - b * BLOCK
            hi = min(start + n, (b + 1) * BLOCK) - b * BLOCK
            z = mu[comp[lo:hi]].astype(np.float32) + 0.6 * eps[lo:hi]
            x = self.s * (z @ w32) + self.m + self.sigma * eta[lo:hi]
            if self.integer:
                x = np.clip(np.rint(x), 0, 255)
            if self.normalize:
                x = x / np.maximum(np.linalg.norm(x, axis=1, keepdims=True), 1e-30)
            pos = b * BLOCK + lo - start
            out[pos:pos + hi - lo] = x

        _for_blocks(block, b0, b1)
        return out


def _for_blocks(fn, b0: int, b1: int) -> None:
    """fn(b) for every block b0..b1; blocks are independent Philox streams, so large ranges run on a thread pool
    (numpy releases the GIL while filling) with bit-identical output."""
    nb = b1 - b0 + 1
    if nb <= 1:
        for b in range(b0, b1 + 1):
            fn(b)
        return
    import concurrent.futures
    import os

    with concurrent.futures.ThreadPoolExecutor(max_workers=min(nb, os.cpu_count() or 1, 16)) as ex:
        list(ex.map(fn, range(b0, b1 + 1)))


@dataclasses.dataclass(frozen=True)
class GCL:
    dim: int
    n_clusters: int = 256
    rank: int = 12
    center_std: float = 25.0
    integer: bool = True

    def _model(self, model_seed: int):
        g = _rng(model_seed, _MODEL_STREAM, 1)
        centers = 64.0 + self.center_std * g.standard_normal((self.n_clusters, self.dim))
        bases = np.empty((self.n_clusters, self.rank, self.dim))
        for c in range(self.n_clusters):
            q, _ = np.linalg.qr(g.standard_normal((self.dim, self.rank)))
            bases[c] = q.T
        return centers, bases

    def rows(self, model_seed: int, row_seed: int, start: int, n: int, ood: bool = False) -> np.ndarray:
        centers, bases = self._model(model_seed)
        out = np.empty((n, self.dim), dtype=np.float32)
        pos = 0
        b0, b1 = start // BLOCK, (start + n - 1) // BLOCK if n > 0 else start // BLOCK - 1
        for b in range(b0, b1 + 1):
            g = _rng(row_seed, _ROW_STREAM, b)
            comp = g.integers(0, self.n_clusters, size=BLOCK)
            u = g.standard_normal((BLOCK, self.rank), dtype=np.float32)
            eta = g.standard_normal((BLOCK, self.dim), dtype=np.float32)
            lo = max(start, b * BLOCK) - b * BLOCK
            hi = min(start + n, (b + 1) * BLOCK) - b * BLOCK
            c = comp[lo:hi]
            x = centers[c] + 40.0 * np.einsum("nr,nrd->nd", u[lo:hi], bases[c]) + 4.0 * eta[lo:hi]
            if self.integer:
                x = np.clip(np.rint(x), 0, 255)
            out[pos:pos + hi - lo] = x
            pos += hi - lo
        return out


# ---- configs (BASELINE.json "configs", shapes per SURVEY.md §8(d) table) ------------------------------
CONFIGS = {
    "C1": dict(workload="C1: 10K x d128 G-LM integer, R=32, 100 queries, k=10, L2",
               n=10_000, dim=128, degree=32, nq=100, k=10, metric=0,
               gen=GLM(dim=128, ell=32, s=30.0, m=64.0, sigma=2.0, integer=True), ood=False),
    "C2": dict(workload="C2: SIFT1M-shaped 1M x d128 fp32 (integer-valued G-LM), R=64, 10K-query batch, k=10, L2",
               n=1_000_000, dim=128, degree=64, nq=10_000, k=10, metric=0,
               gen=GLM(dim=128, ell=32, s=30.0, m=64.0, sigma=2.0, integer=True), ood=False),
    # SURVEY §8(d) C2 "second curve on G-CL (1024 clusters)": the stress generator at C2's shape
    "C2G": dict(workload="C2G: C2 shape (1M x d128 integer-valued, R=64, 10K queries, L2) on the G-CL stress generator "
                         "(1024 clusters, rank-12 subspaces)",
                n=1_000_000, dim=128, degree=64, nq=10_000, k=10, metric=0,
                gen=GCL(dim=128, n_clusters=1024), ood=False),
    "C3": dict(workload="C3: Deep10M-shaped 10M x d96 unit-norm G-LM, R=64, 10K queries, streaming 1% ins/del",
               n=10_000_000, dim=96, degree=64, nq=10_000, k=10, metric=0,
               gen=GLM(dim=96, ell=24, s=1.0, m=0.0, sigma=0.05, normalize=True), ood=False),
    "C4": dict(workload="C4: Text2Image-shaped 10M x d200 IP, OOD queries, sliding window",
               n=10_000_000, dim=200, degree=64, nq=10_000, k=10, metric=1,
               gen=GLM(dim=200, ell=32, s=1.0, m=0.0, sigma=0.05), ood=True),
    "C5": dict(workload="C5: Deep100M-shaped 100M x d96, 8 logical shards",
               n=100_000_000, dim=96, degree=64, nq=10_000, k=10, metric=0,
               gen=GLM(dim=96, ell=24, s=1.0, m=0.0, sigma=0.05, normalize=True), ood=False, shards=8),
}
DATA_SEED, QUERY_SEED, INDEX_SEED = 1, 2, 42


def config_spec(name: str) -> dict:
    return dict(CONFIGS[name])


def base_rows(name: str, start: int = 0, n: Optional[int] = None, model_seed: int = DATA_SEED,
              row_seed: int = DATA_SEED) -> np.ndarray:
    c = CONFIGS[name]
    n = c["n"] - start if n is None else n
    return c["gen"].rows(model_seed, row_seed, start, n)


def query_rows(name: str, n: Optional[int] = None, model_seed: int = DATA_SEED,
               row_seed: int = QUERY_SEED) -> np.ndarray:
    c = CONFIGS[name]
    n = c["nq"] if n is None else n
    return c["gen"].rows(model_seed, row_seed, 0, n, ood=c.get("ood", False))


def int_rows(n: int, dim: int, seed: int, lo: int = 0, hi: int = 256) -> np.ndarray:
    """Uniform integer-valued fp32 rows in [lo, hi) (tiny parity / pin cases)."""
    return _rng(seed, _ROW_STREAM, 0xFFFF).integers(lo, hi, size=(n, dim)).astype(np.float32)


def random_graph(n: int, degree: int, seed: int, n_targets: Optional[int] = None) -> np.ndarray:
    """A random fixed-degree adjacency (uint32 [n][degree]): distinct out-neighbours, no self loops,
    sentinel 0xFFFFFFFF padding when fewer than `degree` targets exist. Structure only, no geometry."""
    n_targets = n if n_targets is None else n_targets
    g = _rng(seed, _ROW_STREAM, 0xFFFE)
    out = np.full((n, degree), 0xFFFFFFFF, dtype=np.uint32)
    for v in range(n):
        pool = n_targets - (1 if v < n_targets else 0)
        take = min(degree, pool)
        pick = g.choice(pool, size=take, replace=False)
        if v < n_targets:
            pick = np.where(pick >= v, pick + 1, pick)
        out[v, :take] = pick
    return out


def random_tombstones(n: int, frac: float, seed: int) -> np.ndarray:
    g = _rng(seed, _ROW_STREAM, 0xFFFD)
    m = int(round(n * frac))
    return np.sort(g.choice(n, size=m, replace=False)).astype(np.uint32)


def pack_tomb(ids, capacity: int) -> np.ndarray:
    """Pack a set of deleted ids into the bitset layout of include/svf.h (bit id%32 of word id/32)."""
    words = np.zeros((capacity + 31) // 32, dtype=np.uint32)
    ids = np.asarray(ids, dtype=np.int64)
    np.bitwise_or.at(words, ids // 32, (np.uint32(1) << (ids % 32).astype(np.uint32)))
    return words
