"""Seeded synthetic graphs with the shapes of BASELINE.json's five configurations, plus the reference's
binary graph snapshot format ("GEMP", /root/reference/proj/src/graph.cpp:141-170).

All randomness comes from a counter-based splitmix64 stream evaluated with numpy uint64 arithmetic, so a
(config, seed) pair produces the same edge list on every machine.  Graphs are undirected, loop-free,
deduplicated, ids 0..n-1, edges in generation order (first occurrence kept).
"""
from __future__ import annotations

import struct

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _finalize(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class Stream:
    """splitmix64 counter stream: draw i is finalize(key + (i+1) * golden)."""

    def __init__(self, seed: int, tag: int = 0):
        with np.errstate(over="ignore"):
            self.key = _finalize(np.array([seed], np.uint64) * _GOLDEN + np.uint64(tag) * _M1 + _GOLDEN)[0]
        self.pos = 0

    def u64(self, count: int) -> np.ndarray:
        idx = np.arange(self.pos + 1, self.pos + 1 + count, dtype=np.uint64)
        self.pos += count
        with np.errstate(over="ignore"):
            return _finalize(self.key + idx * _GOLDEN)

    def uniform(self, count: int) -> np.ndarray:
        return (self.u64(count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def below(self, count: int, bound: int) -> np.ndarray:
        return (self.uniform(count) * bound).astype(np.int64)


def _canonical(n: int, a: np.ndarray, b: np.ndarray):
    """Drops loops, merges duplicate undirected edges, keeps first-occurrence order and orientation."""
    a = a.astype(np.int64)
    b = b.astype(np.int64)
    keep = a != b
    a, b = a[keep], b[keep]
    key = np.minimum(a, b) * np.int64(n) + np.maximum(a, b)
    _, first = np.unique(key, return_index=True)
    first.sort()
    return a[first].astype(np.uint32), b[first].astype(np.uint32)


def sbm_equal(n=3000, blocks=6, p_in=0.02, p_out=0.0005, seed=1):
    """Config 1: stochastic block model with equal blocks (Bernoulli per vertex pair)."""
    rng = Stream(seed, 1)
    size = n // blocks
    block = np.minimum(np.arange(n) // size, blocks - 1)
    src, dst = [], []
    for u0 in range(0, n, 512):  # row panels keep memory flat
        rows = np.arange(u0, min(n, u0 + 512))
        cols = np.arange(n)
        p = np.where(block[rows][:, None] == block[cols][None, :], p_in, p_out)
        hit = (rng.uniform(rows.size * n).reshape(rows.size, n) < p) & (cols[None, :] > rows[:, None])
        r, c = np.nonzero(hit)
        src.append(rows[r])
        dst.append(c)
    s, d = _canonical(n, np.concatenate(src), np.concatenate(dst))
    return n, s, d


def barabasi_albert(n=100_000, m=8, seed=2):
    """Config 2: preferential attachment, m edges per new vertex, seeded from an (m+1)-clique."""
    rng = Stream(seed, 2)
    ends = np.empty(2 * (m * (m + 1) // 2 + m * (n - m - 1)), np.int64)
    src, dst = [], []
    fill = 0
    for i in range(m + 1):
        for j in range(i + 1, m + 1):
            src.append(i)
            dst.append(j)
            ends[fill], ends[fill + 1] = i, j
            fill += 2
    draws = rng.uniform(4 * m * (n - m - 1))
    cursor = 0
    src_new = np.empty(m * (n - m - 1), np.int64)
    dst_new = np.empty(m * (n - m - 1), np.int64)
    out = 0
    for v in range(m + 1, n):
        chosen = set()
        while len(chosen) < m:
            if cursor == draws.size:
                draws = rng.uniform(4 * m * 1024)
                cursor = 0
            chosen.add(int(ends[int(draws[cursor] * fill)]))
            cursor += 1
        for u in chosen:
            src_new[out], dst_new[out] = u, v
            ends[fill], ends[fill + 1] = u, v
            fill += 2
            out += 1
    s, d = _canonical(n, np.concatenate([np.array(src, np.int64), src_new[:out]]),
                      np.concatenate([np.array(dst, np.int64), dst_new[:out]]))
    return n, s, d


def sbm_dirichlet(n=200_000, blocks=10, alpha=2, expected_degree=20, intra=0.8, seed=3):
    """Config 3: block sizes ~ Dirichlet(alpha) (alpha integer: sums of exponentials), n*deg/2 edges,
    a fraction `intra` of them inside the source vertex's block."""
    rng = Stream(seed, 3)
    gam = -np.log(1.0 - rng.uniform(blocks * alpha)).reshape(blocks, alpha).sum(axis=1)
    sizes = np.maximum(1, np.floor(gam / gam.sum() * n).astype(np.int64))
    sizes[-1] += n - sizes.sum()
    starts = np.concatenate([[0], np.cumsum(sizes)])
    block_of = np.repeat(np.arange(blocks), sizes)
    m_total = n * expected_degree // 2
    u = rng.below(m_total, n)
    is_intra = rng.uniform(m_total) < intra
    bu = block_of[u]
    v_in = starts[bu] + (rng.uniform(m_total) * sizes[bu]).astype(np.int64)
    # inter-block partner: uniform over the vertices outside u's block
    off = (rng.uniform(m_total) * (n - sizes[bu])).astype(np.int64)
    v_out = np.where(off < starts[bu], off, off + sizes[bu])
    v = np.where(is_intra, v_in, v_out)
    s, d = _canonical(n, u, v)
    return n, s, d


def rmat(scale=20, edge_factor=16, abcd=(0.57, 0.19, 0.19, 0.05), seed=4, device=None):
    """Configs 4-5: R-MAT, 2^scale vertices, edge_factor * 2^scale generated edges, then symmetrised
    (undirected), loop-free and deduplicated.  With `device` (a torch CUDA device) the same splitmix64 stream
    and the same first-occurrence rule are evaluated with torch, which turns the minutes of numpy work at
    scale 24 into seconds; both paths produce the identical edge list."""
    if device is not None:
        return _rmat_torch(scale, edge_factor, abcd, seed, device)
    rng = Stream(seed, 4)
    n = 1 << scale
    count = edge_factor * n
    a, b, c, _ = abcd
    src = np.zeros(count, np.int64)
    dst = np.zeros(count, np.int64)
    for level in range(scale):
        r = rng.uniform(count)
        src_bit = r >= a + b                       # quadrants c, d
        dst_bit = ((r >= a) & (r < a + b)) | (r >= a + b + c)  # quadrants b, d
        src |= src_bit.astype(np.int64) << level
        dst |= dst_bit.astype(np.int64) << level
    s, d = _canonical(n, src, dst)
    return n, s, d


def _rmat_torch(scale, edge_factor, abcd, seed, device):
    import torch

    def lsr(z, k):  # logical shift right on int64 bit patterns
        return (z >> k) & ((1 << (64 - k)) - 1)

    def finalize(z):
        z = (z ^ lsr(z, 30)) * _as_i64(0xBF58476D1CE4E5B9)
        z = (z ^ lsr(z, 27)) * _as_i64(0x94D049BB133111EB)
        return z ^ lsr(z, 31)

    key = _as_i64(int(Stream(seed, 4).key))
    golden = _as_i64(0x9E3779B97F4A7C15)
    n = 1 << scale
    count = edge_factor * n
    a, b, c, _ = abcd
    src = torch.zeros(count, dtype=torch.int64, device=device)
    dst = torch.zeros(count, dtype=torch.int64, device=device)
    piece = 1 << 26
    for level in range(scale):
        for lo in range(0, count, piece):
            hi = min(count, lo + piece)
            idx = torch.arange(level * count + lo + 1, level * count + hi + 1, dtype=torch.int64, device=device)
            r = lsr(finalize(key + idx * golden), 11).to(torch.float64) * 2.0 ** -53
            src[lo:hi] |= (r >= a + b).to(torch.int64) << level
            dst[lo:hi] |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).to(torch.int64) << level
            del idx, r
    keep = src != dst
    src, dst = src[keep], dst[keep]
    ekey = torch.minimum(src, dst) * n + torch.maximum(src, dst)
    order = torch.sort(ekey, stable=True).indices
    sorted_key = ekey[order]
    is_first = torch.ones_like(sorted_key, dtype=torch.bool)
    is_first[1:] = sorted_key[1:] != sorted_key[:-1]
    first = torch.sort(order[is_first]).values
    s = src[first].to(torch.int32).cpu().numpy().view(np.uint32)
    d = dst[first].to(torch.int32).cpu().numpy().view(np.uint32)
    return n, np.ascontiguousarray(s), np.ascontiguousarray(d)


def _as_i64(v: int) -> int:
    return v - (1 << 64) if v >= (1 << 63) else v


CONFIGS = {
    # name: (generator, kwargs, dim, negatives per vertex, iterations, init rule, init std)
    "c1": (sbm_equal, dict(n=3000, blocks=6, p_in=0.02, p_out=0.0005, seed=1), 2, 5, 200, "uniform_pm1", 0.0),
    "c2": (barabasi_albert, dict(n=100_000, m=8, seed=2), 2, 10, 500, "uniform_pm1", 0.0),
    "c3": (sbm_dirichlet, dict(n=200_000, blocks=10, alpha=2, expected_degree=20, intra=0.8, seed=3), 64, 10, 200,
           "normal", 0.01),
    "c4": (rmat, dict(scale=20, edge_factor=16, seed=4), 128, 20, 100, "normal", 0.01),
    "c5": (rmat, dict(scale=24, edge_factor=16, seed=5), 128, 20, 50, "normal", 0.01),
}


def make_config(name: str, device=None):
    """Returns (n, src, dst, dim, negatives, iterations, init_rule, init_std) for BASELINE config `name`.
    `device` (torch CUDA device) accelerates the R-MAT configurations; the graph is the same either way."""
    gen, kwargs, dim, k, iters, init, std = CONFIGS[name]
    if gen is rmat and device is not None:
        kwargs = dict(kwargs, device=device)
    n, s, d = gen(**kwargs)
    return n, s, d, dim, k, iters, init, std


# ---- the reference's snapshot format (graph.cpp:141-170): "GEMP", u32 n, u64 m, src[m], dst[m], LE ----

def save_snapshot(path: str, n: int, src: np.ndarray, dst: np.ndarray) -> None:
    with open(path, "wb") as f:
        f.write(b"GEMP")
        f.write(struct.pack("<IQ", n, len(src)))
        f.write(np.ascontiguousarray(src, "<u4").tobytes())
        f.write(np.ascontiguousarray(dst, "<u4").tobytes())


def load_snapshot(path: str):
    with open(path, "rb") as f:
        if f.read(4) != b"GEMP":
            raise ValueError("bad snapshot magic")
        head = f.read(12)
        if len(head) != 12:
            raise ValueError("truncated snapshot")
        n, m = struct.unpack("<IQ", head)
        if m == 0:
            raise ValueError("snapshot holds no edges")
        if m > n * (n - 1) // 2:
            raise ValueError("snapshot edge count exceeds pair count")
        src = np.frombuffer(f.read(4 * m), "<u4")
        dst = np.frombuffer(f.read(4 * m), "<u4")
        if src.size != m or dst.size != m:
            raise ValueError("truncated snapshot")
    if (src >= n).any() or (dst >= n).any() or (src == dst).any():
        raise ValueError("snapshot edge out of range")
    return n, src.astype(np.uint32), dst.astype(np.uint32)
