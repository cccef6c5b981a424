"""Seeded synthetic inputs shaped like the paper's workloads.

Used by both the CUDA-path tests and the oracle tests, and by bench.py.  This
module holds no arithmetic of the method itself: it only draws supports and
values.  Recipes (BASELINE.json configs):

* uniform supports: exactly k distinct indices per rank drawn uniformly from
  [0, N) ("k indices out of N are selected uniformly at random at each node
  and are assigned a random value"), values N(0,1) fp32, or
  integers in [-1024, 1024] \\ {0} when sums must be exact in fp32;
* Gaussian gradient vectors (top-k feed, config 3): x ~ N(0,1) fp32;
* clustered LR gradients (config 5): per rank a batch of 1000 samples with
  100 binary features each; feature ids from Zipf(1.1)-ranked 256-wide blocks
  of a random block permutation plus a uniform offset; g_j = sum over samples
  touching j of (sigmoid(0) - y), y ~ Bernoulli(0.5) -> values in Z/2.

Every draw uses numpy's PCG64 seeded with (seed * 1_000_003 + rank).
"""
from __future__ import annotations

import numpy as np

SEED_STRIDE = 1_000_003


def rng_for(seed: int, rank: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed * SEED_STRIDE + rank))


def k_for_density(N: int, d: float) -> int:
    """k = floor(d*N) (R-23)."""
    return int(np.floor(d * N))


def _distinct_sorted(rng: np.random.Generator, N: int, k: int) -> np.ndarray:
    if k > N:
        raise ValueError("k > N")
    if k == 0:
        return np.zeros(0, np.uint32)
    if k * 4 >= N:
        sel = rng.permutation(N)[:k]
    else:
        # rejection on a boolean mask: exact k distinct uniform indices
        taken = np.zeros(N, dtype=bool)
        out = np.empty(0, np.int64)
        need = k
        while need > 0:
            cand = rng.integers(0, N, size=int(need * 1.1) + 16)
            cand = cand[~taken[cand]]
            cand = np.unique(cand)
            rng.shuffle(cand)
            cand = cand[:need]
            taken[cand] = True
            out = np.concatenate([out, cand])
            need = k - len(out)
        sel = out
    return np.sort(sel).astype(np.uint32)


def values(rng: np.random.Generator, n: int, kind: str = "normal") -> np.ndarray:
    if kind == "normal":
        return rng.standard_normal(n, dtype=np.float32)
    if kind == "normal64":   # fp64 values: full 53-bit mantissas
        return rng.standard_normal(n, dtype=np.float64)
    if kind == "int":
        v = rng.integers(1, 1025, size=n)
        s = rng.integers(0, 2, size=n) * 2 - 1
        return (v * s).astype(np.float32)
    if kind == "ones":
        return np.ones(n, np.float32)
    raise ValueError(kind)


def uniform_streams(P: int, N: int, k, seed: int = 0, kind: str = "normal"):
    """P per-rank streams with exactly k[i] (or k) distinct uniform indices."""
    ks = [k] * P if np.isscalar(k) else list(k)
    out = []
    for r in range(P):
        g = rng_for(seed, r)
        idx = _distinct_sorted(g, N, int(ks[r]))
        out.append((idx, values(g, len(idx), kind)))
    return out


def identical_streams(P: int, N: int, k: int, seed: int = 0, kind: str = "int"):
    """Fully overlapping supports H_i = H_j (the RD lower-bound case)."""
    g = rng_for(seed, 0)
    idx = _distinct_sorted(g, N, k)
    return [(idx.copy(), values(rng_for(seed, r + 1), k, kind)) for r in range(P)]


def disjoint_streams(P: int, N: int, k: int, seed: int = 0, kind: str = "int"):
    """Fully disjoint supports (the RD upper-bound case)."""
    if P * k > N:
        raise ValueError("P*k > N")
    g = rng_for(seed, 0)
    allidx = _distinct_sorted(g, N, P * k)
    perm = g.permutation(P * k)
    out = []
    for r in range(P):
        sel = np.sort(allidx[perm[r * k:(r + 1) * k]])
        out.append((sel.astype(np.uint32), values(rng_for(seed, r + 1), k, kind)))
    return out


def gaussian_vector(N: int, seed: int = 0, rank: int = 0) -> np.ndarray:
    return rng_for(seed, rank).standard_normal(N, dtype=np.float32)


def lr_gradient_streams(P: int, N: int = 3_231_961, samples: int = 1000, feats: int = 100,
                        seed: int = 0, block: int = 256, zipf_a: float = 1.1):
    """Naturally sparse logistic-regression gradients at w = 0 (config 5).

    Returns per-rank (idx, val) with explicit zeros kept (support = every
    feature the batch touches).  Values are exact multiples of 1/2."""
    nblocks = (N + block - 1) // block
    perm = rng_for(seed, 10_000).permutation(nblocks)
    out = []
    for r in range(P):
        g = rng_for(seed, r)
        ranks = g.zipf(zipf_a, size=(samples, feats))
        ranks = np.minimum(ranks - 1, nblocks - 1)
        blk = perm[ranks]
        feat = blk * block + g.integers(0, block, size=(samples, feats))
        feat = np.minimum(feat, N - 1)
        y = g.integers(0, 2, size=samples).astype(np.float64)
        coef = 0.5 - y   # sigmoid(0) - y
        # binary features: each (sample, feature) pair contributes coef once
        keys = np.concatenate([np.unique(feat[s]) for s in range(samples)])
        contrib = np.concatenate([np.full(len(np.unique(feat[s])), coef[s]) for s in range(samples)])
        uniq, inv = np.unique(keys, return_inverse=True)
        gsum = np.zeros(len(uniq), np.float64)
        np.add.at(gsum, inv, contrib)
        out.append((uniq.astype(np.uint32), gsum.astype(np.float32)))
    return out


def lr_dataset(P: int, N: int, samples: int = 1000, feats: int = 100, seed: int = 0, block: int = 256,
               zipf_a: float = 1.1):
    """Per-rank synthetic sparse logistic-regression data with config 5's structure:
    `samples` samples of `feats` binary features, feature blocks of `block` drawn
    Zipf(zipf_a) over a random block permutation, labels y in {0, 1} from a hidden
    sparse model (so the problem is learnable).  Returns [(feat int64[samples, feats], y float32[samples])]."""
    nblocks = (N + block - 1) // block
    perm = rng_for(seed, 10_000).permutation(nblocks)
    w_true = np.zeros(N, np.float64)
    gt = rng_for(seed, 20_000)
    hot = gt.choice(N, size=max(1, N // 50), replace=False)
    w_true[hot] = gt.standard_normal(len(hot)) * 2.0
    out = []
    for r in range(P):
        g = rng_for(seed, r)
        ranks = np.minimum(g.zipf(zipf_a, size=(samples, feats)) - 1, nblocks - 1)
        feat = np.minimum(perm[ranks] * block + g.integers(0, block, size=(samples, feats)), N - 1)
        margin = np.array([w_true[np.unique(f)].sum() for f in feat])
        y = (g.random(samples) < 1.0 / (1.0 + np.exp(-margin))).astype(np.float32)
        out.append((feat.astype(np.int64), y))
    return out
