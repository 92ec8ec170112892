"""Seeded synthetic instances for the five BASELINE.json configurations.

All generators emit canonical CSR directly (rows sorted, symmetric,
deduplicated, no self-loops), bypassing build_graph's validation pass, as the
reference's own WeightedGraph(n, indptr, indices, w) constructor allows
(graph.py:37).  Column indices are int32 (every config has n < 2^31).

  C1  Erdos-Renyi G(1000, p = 10/999), w = 1 - U[0,1) in (0,1], fp64
  C2  assignment conflict graph of a 256x256 assignment (line graph of
      K_{256,256}): 65,536 vertices, degree 510, w ~ U(0,1] drawn in fp32
  C3  Barabasi-Albert n = 200,000, m = 5 (networkx's algorithm: star seed,
      preferential attachment), integer weights U{1..200} stored fp64
  C4  batch of independent G(2000, 16/1999) graphs packed block-diagonally,
      w = 1 - U fp32, per-graph x0 = init_random(2000, [seed, g])
  C5  R-MAT (a,b,c,d) = (.57,.19,.19,.05), edge factor 16, symmetrised and
      deduplicated, w = 1 - U fp32.  The random stream is a counter-based
      hash (splitmix64 of (seed, edge, level)), so the same graph can be
      generated on the GPU at scale 24 and on the CPU at small scales.

fp32 configs draw weights and starts that are exactly representable in
binary32, so the fp64 oracle and the fp32 engine start from identical values.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .dynamics import init_random
from .graph import WeightedGraph


@dataclass
class Instance:
    name: str
    graph: WeightedGraph
    x0: np.ndarray
    dtype: str
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.graph.n

    @property
    def m(self) -> int:
        return self.graph.num_edges


def _canonical(n: int, lo: np.ndarray, hi: np.ndarray, dedup: bool = True) -> tuple[np.ndarray, np.ndarray]:
    """CSR from undirected pairs (lo != hi).  int64 indptr, int32 indices."""
    lo = np.asarray(lo, dtype=np.int64)
    hi = np.asarray(hi, dtype=np.int64)
    a = np.minimum(lo, hi)
    b = np.maximum(lo, hi)
    if dedup:
        key = np.unique(a * np.int64(n) + b)
        a = key // n
        b = key % n
    rows = np.concatenate([a, b])
    cols = np.concatenate([b, a])
    key2 = rows * np.int64(n) + cols
    key2.sort()
    rows = key2 // n
    cols = (key2 % n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    return indptr, cols


def f32_exact(a: np.ndarray) -> np.ndarray:
    """Round to binary32 and back: values both engines see identically."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


# ---------------------------------------------------------------- ER

def er_pairs(n: int, p: float, rng: np.random.Generator) -> tuple[np.ndarray, np.ndarray]:
    """Exact G(n, p) pair sampling by geometric skips over the n(n-1)/2 pairs
    in (u<v) row-major order (same distribution as a Bernoulli mask)."""
    total = n * (n - 1) // 2
    if total == 0 or p <= 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    out = []
    pos = -1
    while True:
        need = int(max(64, (total - pos) * p * 1.1 + 64))
        gaps = rng.geometric(p, size=need).astype(np.int64)
        idx = pos + np.cumsum(gaps)
        keep = idx[idx < total]
        out.append(keep)
        if len(keep) < len(idx):
            break
        pos = int(idx[-1])
    lin = np.concatenate(out)
    # linear index -> (u, v), u < v, row-major over the strict upper triangle
    u = (n - 2 - np.floor(np.sqrt(-8.0 * lin + 4.0 * n * (n - 1) - 7) / 2.0 - 0.5)).astype(np.int64)
    start = u * (2 * n - u - 1) // 2
    # fix rare float rounding at row boundaries
    over = lin < start
    while over.any():
        u[over] -= 1
        start = u * (2 * n - u - 1) // 2
        over = lin < start
    nxt = (u + 1) * (2 * n - u - 2) // 2
    under = lin >= nxt
    while under.any():
        u[under] += 1
        start = u * (2 * n - u - 1) // 2
        nxt = (u + 1) * (2 * n - u - 2) // 2
        under = lin >= nxt
    v = lin - start + u + 1
    return u, v


def c1_er(n: int = 1000, avg_degree: float = 10.0, seed: int = 2605_0001) -> Instance:
    """C1: ER G(n, d/(n-1)) with the reference's triu + uniform-mask
    construction (graph.py:197-200), w = 1 - U[0,1), x0 = init_random."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    pick = rng.random(len(iu)) < avg_degree / (n - 1)
    w = 1.0 - rng.random(n)
    indptr, indices = _canonical(n, iu[pick], ju[pick], dedup=False)
    g = WeightedGraph(n, indptr, indices, w)
    return Instance("C1-er1000", g, init_random(n, [seed, 1]), "fp64",
                    {"avg_degree": avg_degree, "seed": seed})


# ---------------------------------------------------------------- C2

def c2_assignment(k: int = 256, seed: int = 2605_0002) -> Instance:
    """C2: conflict graph of a k x k assignment.  Vertex (i, j) -> k*i + j is
    adjacent to every vertex sharing its row or its column (degree 2(k-1))."""
    n = k * k
    i = np.repeat(np.arange(k, dtype=np.int64), k)
    j = np.tile(np.arange(k, dtype=np.int64), k)
    deg = 2 * (k - 1)
    # sorted neighbour list of (i, j): column part above, row part, column part below
    t = np.arange(k, dtype=np.int64)
    col_part = t[None, :] * k + j[:, None]           # (n, k): k*i' + j
    row_part = i[:, None] * k + t[None, :]           # (n, k): k*i + j'
    col_mask = t[None, :] != i[:, None]
    row_mask = t[None, :] != j[:, None]
    above = np.where(t[None, :] < i[:, None], col_part, -1)
    below = np.where(t[None, :] > i[:, None], col_part, -1)
    rowv = np.where(row_mask, row_part, -1)
    allnb = np.concatenate([above, rowv, below], axis=1)
    allnb = allnb[allnb >= 0].reshape(n, deg)
    del col_mask
    indices = allnb.astype(np.int32).ravel()
    indptr = np.arange(n + 1, dtype=np.int64) * deg
    rng = np.random.default_rng(seed)
    w = (np.float32(1.0) - rng.random(n, dtype=np.float32)).astype(np.float64)
    g = WeightedGraph(n, indptr, indices, w)
    x0 = f32_exact(init_random(n, [seed, 1]))
    return Instance(f"C2-assignment{k}x{k}", g, x0, "fp32", {"k": k, "seed": seed})


# ---------------------------------------------------------------- C3

def barabasi_albert_pairs(n: int, m: int, rng: np.random.Generator) -> tuple[np.ndarray, np.ndarray]:
    """networkx.barabasi_albert_graph's algorithm: a star on m+1 vertices,
    then each new vertex attaches to m distinct targets drawn uniformly from
    the degree-weighted repeated-node list."""
    src = np.empty(m + (n - m - 1) * m, dtype=np.int64)
    dst = np.empty_like(src)
    src[:m] = 0
    dst[:m] = np.arange(1, m + 1)
    repeated = np.empty(2 * len(src), dtype=np.int64)
    repeated[:m] = 0
    repeated[m:2 * m] = np.arange(1, m + 1)
    rlen = 2 * m
    e = m
    batch = rng.random(1 << 20)
    bi = 0
    for source in range(m + 1, n):
        chosen = set()
        while len(chosen) < m:
            if bi == len(batch):
                batch = rng.random(1 << 20)
                bi = 0
            chosen.add(int(repeated[int(batch[bi] * rlen)]))
            bi += 1
        tg = sorted(chosen)
        src[e:e + m] = source
        dst[e:e + m] = tg
        e += m
        repeated[rlen:rlen + m] = tg
        repeated[rlen + m:rlen + 2 * m] = source
        rlen += 2 * m
    return src, dst


def c3_ba(n: int = 200_000, m: int = 5, seed: int = 2605_0003) -> Instance:
    rng = np.random.default_rng(seed)
    s, d = barabasi_albert_pairs(n, m, rng)
    indptr, indices = _canonical(n, s, d)
    w = rng.integers(1, 201, size=n).astype(np.float64)
    g = WeightedGraph(n, indptr, indices, w)
    return Instance(f"C3-ba{n}m{m}", g, init_random(n, [seed, 1]), "fp64", {"m": m, "seed": seed})


# ---------------------------------------------------------------- C4

@dataclass
class Batch:
    """Independent graphs packed block-diagonally into one CSR."""

    instance: Instance
    offsets: np.ndarray  # graph b owns vertices [offsets[b], offsets[b+1])


def c4_batch(graphs: int = 1024, n: int = 2000, avg_degree: float = 16.0, seed: int = 2605_0004,
             first: int = 0) -> Batch:
    """Graphs first..first+graphs-1 of the C4 family, packed.  Each graph has
    its own RNG stream [seed, g], so any shard of the family is reproducible
    on its own (rank r of G takes first = r * graphs)."""
    p = avg_degree / (n - 1)
    los, his, ws, xs = [], [], [], []
    for b in range(graphs):
        gid = first + b
        rng = np.random.default_rng([seed, gid])
        u, v = er_pairs(n, p, rng)
        off = b * n
        los.append(u + off)
        his.append(v + off)
        ws.append(np.float32(1.0) - rng.random(n, dtype=np.float32))
        xs.append(f32_exact(init_random(n, [seed, gid, 1])))
    N = graphs * n
    indptr, indices = _canonical(N, np.concatenate(los), np.concatenate(his), dedup=False)
    w = np.concatenate(ws).astype(np.float64)
    g = WeightedGraph(N, indptr, indices, w)
    inst = Instance(f"C4-batch{graphs}x{n}", g, np.concatenate(xs), "fp32",
                    {"graphs": graphs, "n_per_graph": n, "first": first, "seed": seed})
    return Batch(inst, np.arange(graphs + 1, dtype=np.int64) * n)


# ---------------------------------------------------------------- C5

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def rmat_pairs(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
               seed: int = 2605_0005, chunk: int = 1 << 22) -> tuple[np.ndarray, np.ndarray]:
    """Counter-based R-MAT: level l of edge e uses u = splitmix64(seed*2^40 +
    e*64 + l) (top 53 bits / 2^53).  Bit-identical to the GPU generator."""
    ne = (1 << scale) * edge_factor
    srcs, dsts = [], []
    ab, abc = a + b, a + b + c
    base = np.uint64(seed) << np.uint64(40)
    for e0 in range(0, ne, chunk):
        e = np.arange(e0, min(ne, e0 + chunk), dtype=np.uint64)
        s = np.zeros(len(e), dtype=np.int64)
        d = np.zeros(len(e), dtype=np.int64)
        for lvl in range(scale):
            with np.errstate(over="ignore"):
                h = splitmix64(base + e * np.uint64(64) + np.uint64(lvl))
            u = (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
            rbit = (u >= ab).astype(np.int64)
            cbit = ((u >= a) & (u < ab)) | (u >= abc)
            s = (s << 1) | rbit
            d = (d << 1) | cbit.astype(np.int64)
        srcs.append(s)
        dsts.append(d)
    return np.concatenate(srcs), np.concatenate(dsts)


def hash_uniform_f32(seed: int, n: int, stream: int) -> np.ndarray:
    """Counter-based U[0,1) in binary32 steps of 2^-24."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64((np.uint64(seed) << np.uint64(40)) ^ (np.uint64(stream) << np.uint64(36)) ^ i)
    return (h >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0)


def c5_rmat(scale: int = 16, edge_factor: int = 16, seed: int = 2605_0005) -> Instance:
    n = 1 << scale
    s, d = rmat_pairs(scale, edge_factor, seed=seed)
    keep = s != d
    indptr, indices = _canonical(n, s[keep], d[keep])
    w = 1.0 - hash_uniform_f32(seed, n, 1)
    x0 = f32_exact(init_random(n, [seed, 1]))
    g = WeightedGraph(n, indptr, indices, w)
    return Instance(f"C5-rmat{scale}", g, x0, "fp32",
                    {"scale": scale, "edge_factor": edge_factor, "seed": seed,
                     "sampled_edges": int(len(s)), "unique_edges": int(len(indices) // 2)})


def rmat_csr_gpu(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
                 seed: int = 2605_0005, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """The R-MAT of rmat_pairs + _canonical, generated, deduplicated and
    turned into CSR on the GPU (csrc/gn_gen.cu); bitwise the CPU result."""
    import ctypes

    from . import _engine as E

    nnz = ctypes.c_int64()
    pp, pc = ctypes.c_void_p(), ctypes.c_void_p()
    E.check(E.lib().gn_gen_rmat(scale, edge_factor, a, b, c, seed, device, ctypes.byref(nnz), ctypes.byref(pp),
                                ctypes.byref(pc)))
    n = 1 << scale
    try:
        indptr = np.ctypeslib.as_array(ctypes.cast(pp, ctypes.POINTER(ctypes.c_int64)), shape=(n + 1,)).copy()
        indices = (np.ctypeslib.as_array(ctypes.cast(pc, ctypes.POINTER(ctypes.c_int32)), shape=(nnz.value,)).copy()
                   if nnz.value else np.zeros(0, np.int32))
    finally:
        E.lib().gn_free_host(pp)
        E.lib().gn_free_host(pc)
    return indptr, indices


def c5_rmat_gpu(scale: int = 24, edge_factor: int = 16, seed: int = 2605_0005, device: int = 0) -> Instance:
    """C5 at full scale: the graph of c5_rmat(scale) built on the GPU."""
    n = 1 << scale
    indptr, indices = rmat_csr_gpu(scale, edge_factor, seed=seed, device=device)
    w = 1.0 - hash_uniform_f32(seed, n, 1)
    x0 = f32_exact(init_random(n, [seed, 1]))
    g = WeightedGraph(n, indptr, indices, w)
    return Instance(f"C5-rmat{scale}", g, x0, "fp32",
                    {"scale": scale, "edge_factor": edge_factor, "seed": seed, "sampled_edges": n * edge_factor,
                     "unique_edges": int(len(indices) // 2), "generated_on": "gpu"})


CONFIGS = {
    "C1": c1_er,
    "C2": c2_assignment,
    "C3": c3_ba,
    "C5": c5_rmat,
}
