"""Seeded synthetic inputs shaped like the paper's workloads (no CKKS arithmetic here).

This is the ONE module shared by the product path, the oracle-based tests and bench.py:
it only draws float64 feature vectors with numpy.  The paper's timing workload is
6,144 IJB-C face embeddings, d = 128, from a ResNet-18/ArcFace extractor (PAPER.md:533,
553-556); the dataset and weights are not available, so seeded unit-norm Gaussian
vectors (uniform on the sphere, like L2-normalised ArcFace embeddings) stand in with
the same count and dimension.  Configs follow
BASELINE.json `configs`.
"""
import numpy as np

DATA_SEED_BASE = 240806167 * 10


def _unit(x):
    return x / np.linalg.norm(x, axis=-1, keepdims=True)


CONFIGS = {
    # id: (d, n_templates, default p, p sweep, n_queries)
    1: dict(d=16, n=256, p=1, p_sweep=(1,), nq=1),
    2: dict(d=128, n=6144, p=8, p_sweep=(1, 2, 4, 8), nq=384),
    3: dict(d=32, n=65536, p=4, p_sweep=(1, 2, 4), nq=64),
    4: dict(d=128, n=1048576, p=8, p_sweep=(8,), nq=256),
    5: dict(d=512, n=4194304, p=16, p_sweep=(4, 8, 16), nq=1024),
}


def templates(cfg, n=None, first=0):
    """Templates [n][d] float64, unit norm.  Rows are generated in fixed chunks of 65,536
    so any row range is reproducible without drawing the whole database."""
    c = CONFIGS[cfg]
    d = c["d"]
    n = c["n"] - first if n is None else n
    if cfg == 3:
        rng = np.random.default_rng(DATA_SEED_BASE + cfg)
        cent = _unit(rng.standard_normal((4096, d)))
        noise = rng.standard_normal((4096, 16, d)) * 0.1
        allt = _unit(cent[:, None, :] + noise).reshape(-1, d)
        return allt[first:first + n]
    # rows are drawn in fixed chunks of 65,536 (row-major, so the first k rows of a chunk do not
    # depend on how many are drawn); rows past the config's count extend the same stream
    # (weak-scaling shards of bench.py use them)
    CH = 65536
    out = np.empty((n, d))
    row = first
    while row < first + n:
        ch = row // CH
        lo = row - ch * CH
        take = min(CH - lo, first + n - row)
        rng = np.random.default_rng([DATA_SEED_BASE + cfg, ch])
        block = rng.standard_normal((lo + take, d))[lo:]
        out[row - first:row - first + take] = _unit(block)
        row += take
    return out


def template_rows(cfg, rows):
    """templates(cfg, 1, u)[0] for every u in rows (the same values), drawing each 65,536-row chunk
    once up to the last row needed from it."""
    d = CONFIGS[cfg]["d"]
    rows = np.asarray(rows, np.int64)
    out = np.empty((rows.size, d))
    CH = 65536
    for ch in np.unique(rows // CH):
        sel = np.nonzero(rows // CH == ch)[0]
        hi = int((rows[sel] - ch * CH).max()) + 1
        rng = np.random.default_rng([DATA_SEED_BASE + cfg, int(ch)])
        block = _unit(rng.standard_normal((hi, d)))
        out[sel] = block[rows[sel] - ch * CH]
    return out


def queries(cfg, nq=None):
    """Queries [nq][d] float64 unit norm, and the expected genuine template index (-1 = impostor).

    C1: normalise(T[17] + N(0, 0.05^2))                      -> 17
    C2: normalise(T[16 j] + N(0, 0.05^2)), j < 384            -> 16 j
    C3: normalise(c_j + N(0, 0.1^2)) for 64 distinct identities -> identity (template index 16 c_j)
    C4: 128 genuine (random distinct u_j, sigma 0.05) + 128 impostors (fresh unit Gaussian)
    C5: 256 genuine from u = 0 mod 4 + 768 impostors
    """
    c = CONFIGS[cfg]
    d = c["d"]
    nq = c["nq"] if nq is None else nq
    rng = np.random.default_rng(DATA_SEED_BASE + 1000 + cfg)
    if cfg == 1:
        T = templates(1)
        q = _unit(T[17] + rng.standard_normal(d) * 0.05)[None].repeat(nq, 0)
        return q, np.full(nq, 17)
    if cfg == 2:
        T = templates(2)
        idx = 16 * np.arange(nq) % c["n"]
        return _unit(T[idx] + rng.standard_normal((nq, d)) * 0.05), idx
    if cfg == 3:
        rng0 = np.random.default_rng(DATA_SEED_BASE + cfg)
        cent = _unit(rng0.standard_normal((4096, d)))
        ids = rng.choice(4096, size=nq, replace=False)
        return _unit(cent[ids] + rng.standard_normal((nq, d)) * 0.1), 16 * ids
    n_gen = nq // 2 if cfg == 4 else nq // 4
    if cfg == 4:
        u = rng.choice(c["n"], size=n_gen, replace=False)
    else:
        u = 4 * rng.choice(c["n"] // 4, size=n_gen, replace=False)
    gen = template_rows(cfg, u) if n_gen else np.zeros((0, d))
    gen = _unit(gen + rng.standard_normal((n_gen, d)) * 0.05)
    imp = _unit(rng.standard_normal((nq - n_gen, d)))
    return np.concatenate([gen, imp]), np.concatenate([u, np.full(nq - n_gen, -1)])


def random_unit(n, d, seed):
    """Generic seeded unit vectors for tests (ragged / edge-case shapes)."""
    return _unit(np.random.default_rng(seed).standard_normal((n, d)))
