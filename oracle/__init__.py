"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the two CPU checkers.

* ``Oracle``  : oracle/_build/libgempe_oracle.so, the plain-C restatement (gempe_oracle.c).
* ``Ref``     : oracle/_ref/libgempe_ref.so, the UNMODIFIED reference compiled from
  /root/reference/proj by oracle/Makefile (absent sources => prebuilt file is used as shipped).

Only tests/, tools/make_golden.py, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libgempe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgempe_ref.so")

BINS = 512
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the checkers (the C restatement always; _ref only when the sources are mounted)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


class GoTable(C.Structure):
    _fields_ = [("knots", C.c_double * 17), ("a", C.c_double * 16), ("b", C.c_double * 16),
                ("c", C.c_double * 16), ("lo", C.c_double), ("hi", C.c_double),
                ("odd_mirror", C.c_int)]


class GoFastMath(C.Structure):
    _fields_ = [("erf", GoTable), ("ratio", GoTable)]


def _table_from_flat(flat, odd):
    t = GoTable()
    flat = [float(v) for v in flat]
    for i in range(17):
        t.knots[i] = flat[i]
    for i in range(16):
        t.a[i] = flat[17 + i]
        t.b[i] = flat[33 + i]
        t.c[i] = flat[49 + i]
    t.lo, t.hi = flat[65], flat[66]
    t.odd_mirror = int(odd)
    return t


def fastmath_from_flat(erf_flat, ratio_flat) -> GoFastMath:
    """Tables in the flat layout knots[17] a[16] b[16] c[16] lo hi (67 doubles each)."""
    fm = GoFastMath()
    fm.erf = _table_from_flat(erf_flat, 1)
    fm.ratio = _table_from_flat(ratio_flat, 0)
    return fm


class Oracle:
    """The C restatement.  Method names follow gempe_oracle.h."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = self.lib = C.CDLL(ORACLE_SO)
        L.go_splitmix64.restype = C.c_uint64
        L.go_splitmix64.argtypes = [C.c_uint64]
        L.go_mix_seed.restype = C.c_uint64
        L.go_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.go_expand_seed32.restype = C.c_uint32
        L.go_expand_seed32.argtypes = [C.c_uint64] * 4
        L.go_lcg_next.restype = C.c_uint32
        L.go_lcg_next.argtypes = [C.c_uint32]
        L.go_lane_uniform_index.restype = C.c_uint32
        L.go_lane_uniform_index.argtypes = [C.c_uint32, C.c_uint32]
        L.go_pair_hash.restype = C.c_uint32
        L.go_pair_hash.argtypes = [C.c_uint32] * 4
        L.go_hash_bits.restype = C.c_int
        L.go_hash_bits.argtypes = [C.c_uint64, C.c_int]
        L.go_hash_build.restype = None
        L.go_hash_build.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_int, u8p]
        L.go_sample_one.restype = C.c_int
        L.go_sample_one.argtypes = [u8p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.go_random_relabel.restype = None
        L.go_random_relabel.argtypes = [C.c_uint32, C.c_uint64, u32p]
        L.go_init_embedding.restype = None
        L.go_init_embedding.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p]
        L.go_table_eval.restype = C.c_double
        L.go_table_eval.argtypes = [C.POINTER(GoTable), C.c_double]
        L.go_gauss_over_erfc.restype = C.c_double
        L.go_gauss_over_erfc.argtypes = [C.c_double]
        L.go_ratio_fast.restype = C.c_double
        L.go_ratio_fast.argtypes = [C.POINTER(GoFastMath), C.c_double]
        L.go_parabola.restype = None
        L.go_parabola.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int,
                                  C.POINTER(GoFastMath), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]
        L.go_hist_bin.restype = C.c_int
        L.go_hist_bin.argtypes = [C.c_double]
        for name in ("go_histogram_objective", "go_histogram_objective_dsigma"):
            f = getattr(L, name)
            f.restype = C.c_double
            f.argtypes = [u64p, u64p, C.c_double, C.c_double, C.c_double]
        L.go_optimize_sigma.restype = C.c_double
        L.go_optimize_sigma.argtypes = [u64p, u64p, C.c_double, C.c_double, C.POINTER(C.c_int)]
        L.go_iterate.restype = C.c_int
        L.go_iterate.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_uint32, f32p, C.c_int,
                                 C.c_uint32, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                 C.POINTER(GoFastMath), C.c_void_p, C.c_uint32, C.c_void_p,
                                 f64p, f64p, u64p, u64p, f32p, u32p, C.POINTER(C.c_uint64)]

        L.go_pairs_accumulate.restype = None
        L.go_pairs_accumulate.argtypes = [C.c_uint32, C.c_void_p, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                          C.c_uint64, u32p, u32p, C.c_int, C.c_double, C.c_double,
                                          C.POINTER(GoFastMath), f64p, f64p, C.c_void_p]

    # -- thin conveniences -------------------------------------------------------------------
    def hash_build(self, n, src, dst, bits_override=0):
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        bits = self.lib.go_hash_bits(len(src), int(bits_override))
        table = np.zeros(1 << bits, np.uint8)
        self.lib.go_hash_build(n, len(src), src, dst, bits, table)
        return table

    def random_relabel(self, n, seed):
        fwd = np.empty(n, np.uint32)
        self.lib.go_random_relabel(n, seed, fwd)
        return fwd

    def init_embedding(self, n, dim, seed):
        out = np.empty((n, dim), np.float32)
        self.lib.go_init_embedding(n, dim, seed, out)
        return out

    def parabola(self, delta, mu, sigma, is_edge, fm=None):
        d, w = C.c_double(), C.c_double()
        self.lib.go_parabola(delta, mu, sigma, int(is_edge), C.byref(fm) if fm is not None else None,
                             C.byref(d), C.byref(w))
        return d.value, w.value

    def optimize_sigma(self, he, hn, nonedge_weight, mu):
        steps = C.c_int()
        s = self.lib.go_optimize_sigma(np.ascontiguousarray(he, np.uint64),
                                       np.ascontiguousarray(hn, np.uint64), nonedge_weight, mu,
                                       C.byref(steps))
        return s, steps.value

    def subset_yz(self, n, x, subset, edge_pairs, sample_pairs, mu, sigma, fm):
        """(y, z) of the vertices in `subset` from explicit pair lists (go_pairs_accumulate): edge_pairs /
        sample_pairs = (a, b) uint32 arrays holding every pair that touches a subset vertex exactly once."""
        x = np.ascontiguousarray(x, np.float32)
        dim = x.shape[1]
        subset = np.asarray(subset, np.int64)
        index = np.full(n, -1, np.int32)
        index[subset] = np.arange(subset.size, dtype=np.int32)
        y = np.zeros((subset.size, dim), np.float64)
        z = np.zeros(subset.size, np.float64)
        for (a, b), is_edge in ((edge_pairs, 1), (sample_pairs, 0)):
            a = np.ascontiguousarray(a, np.uint32)
            b = np.ascontiguousarray(b, np.uint32)
            self.lib.go_pairs_accumulate(dim, x.ctypes.data_as(C.c_void_p), index, a.size, a, b, is_edge, mu, sigma,
                                         C.byref(fm) if fm is not None else None, y, z, None)
        return y, z

    def iterate(self, n, src, dst, x, neg_mode, k, seed, it, mu, sigma, fm, table,
                forced_partners=None):
        """One Jacobi round in double.  Returns dict(rc, y, z, hist_edge, hist_nonedge, x_next,
        partners, draws)."""
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        x = np.ascontiguousarray(x, np.float32)
        dim = x.shape[1]
        m = len(src)
        slots = 2 * m if neg_mode == 0 else n * k
        y = np.zeros((n, dim), np.float64)
        z = np.zeros(n, np.float64)
        he = np.zeros(BINS, np.uint64)
        hn = np.zeros(BINS, np.uint64)
        xn = np.zeros((n, dim), np.float32)
        partners = np.zeros(max(slots, 1), np.uint32)
        draws = C.c_uint64(0)
        forced = None
        if forced_partners is not None:
            forced_arr = np.ascontiguousarray(forced_partners, np.uint32)
            forced = forced_arr.ctypes.data_as(C.c_void_p)
        tab = np.ascontiguousarray(table, np.uint8)
        rc = self.lib.go_iterate(n, m, src, dst, dim, x, neg_mode, k, seed, it, mu, sigma,
                                 C.byref(fm) if fm is not None else None,
                                 tab.ctypes.data_as(C.c_void_p), len(tab), forced, y, z, he, hn,
                                 xn, partners, C.byref(draws))
        return dict(rc=rc, y=y, z=z, hist_edge=he, hist_nonedge=hn, x_next=xn,
                    partners=partners[:slots], draws=draws.value)


class Ref:
    """The unmodified reference behind oracle/ref_shim.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = self.lib = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_expand_seed32.restype = C.c_uint32
        L.ref_expand_seed32.argtypes = [C.c_uint64] * 4
        L.ref_lane_uniform_index.restype = C.c_uint32
        L.ref_lane_uniform_index.argtypes = [C.c_uint32, C.c_uint32]
        L.ref_pair_hash.restype = C.c_uint32
        L.ref_pair_hash.argtypes = [C.c_uint32] * 4
        L.ref_random_relabel.argtypes = [C.c_uint32, C.c_uint64, u32p]
        L.ref_init_embedding.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p]
        L.ref_hash_build.restype = C.c_void_p
        L.ref_hash_build.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_int]
        L.ref_hash_free.argtypes = [C.c_void_p]
        L.ref_hash_size.restype = C.c_uint32
        L.ref_hash_size.argtypes = [C.c_void_p]
        L.ref_hash_bits.argtypes = [C.c_void_p]
        L.ref_hash_occupied.restype = C.c_uint64
        L.ref_hash_occupied.argtypes = [C.c_void_p]
        L.ref_hash_probe.argtypes = [C.c_void_p, u32p, u32p, C.c_uint64, u8p]
        L.ref_sample_non_edges.argtypes = [C.c_void_p, C.c_uint32, u32p, u32p, C.c_uint64, u32p,
                                           C.POINTER(C.c_uint64)]
        L.ref_fastmath_table.argtypes = [C.c_int, f64p]
        L.ref_gauss_erfc_ratio.restype = C.c_double
        L.ref_gauss_erfc_ratio.argtypes = [C.c_double, C.c_int]
        L.ref_parabola.restype = None
        L.ref_parabola.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_description_length.restype = C.c_double
        L.ref_description_length.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        L.ref_optimize_sigma.argtypes = [u64p, u64p, C.c_double, C.c_double,
                                         C.POINTER(C.c_double), C.POINTER(C.c_int)]
        for name in ("ref_histogram_objective", "ref_histogram_objective_dsigma"):
            f = getattr(L, name)
            f.restype = C.c_double
            f.argtypes = [u64p, u64p, C.c_double, C.c_double, C.c_double]
        L.ref_engine_create.restype = C.c_void_p
        L.ref_engine_create.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_uint32, C.c_uint32,
                                        C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_int, C.c_uint64]
        L.ref_engine_free.argtypes = [C.c_void_p]
        L.ref_engine_degenerate.argtypes = [C.c_void_p]
        L.ref_engine_iteration.argtypes = [C.c_void_p]
        L.ref_engine_sigma.restype = C.c_double
        L.ref_engine_sigma.argtypes = [C.c_void_p]
        L.ref_engine_hash_size.restype = C.c_uint32
        L.ref_engine_hash_size.argtypes = [C.c_void_p]
        L.ref_engine_work_graph.argtypes = [C.c_void_p, u32p, u32p]
        L.ref_engine_work_coords.argtypes = [C.c_void_p, f32p]
        L.ref_engine_probe.argtypes = [C.c_void_p, u32p, u32p, C.c_uint64, u8p]
        L.ref_engine_iterate.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.c_void_p, C.c_void_p]
        L.ref_engine_set_capture.argtypes = [C.c_void_p, C.c_int]
        L.ref_engine_run.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                     C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_double), C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_double)]
        L.ref_pe_exact.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_uint32, f32p,
                                   C.POINTER(C.c_double)]
        L.ref_pe_sampled.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_uint32, f32p, C.c_int, C.c_uint64,
                                     C.POINTER(C.c_double)]
        L.ref_load_edge_list.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.ref_write_embedding_tsv.restype = C.c_long
        L.ref_write_embedding_tsv.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_long]
        L.ref_save_graph_snapshot.restype = C.c_long
        L.ref_save_graph_snapshot.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, C.c_void_p, C.c_long]

    def error(self):
        return self.lib.ref_last_error().decode(errors="replace")

    def fastmath_table(self, which):
        out = np.zeros(67, np.float64)
        odd = self.lib.ref_fastmath_table(which, out)
        return out, odd

    def fastmath(self) -> GoFastMath:
        return fastmath_from_flat(self.fastmath_table(0)[0], self.fastmath_table(2)[0])

    def parabola(self, delta, mu, sigma, is_edge, fast):
        d, w = C.c_double(), C.c_double()
        self.lib.ref_parabola(delta, mu, sigma, int(is_edge), int(fast), C.byref(d), C.byref(w))
        return d.value, w.value

    def optimize_sigma(self, he, hn, nonedge_weight, mu):
        s, steps = C.c_double(), C.c_int()
        rc = self.lib.ref_optimize_sigma(np.ascontiguousarray(he, np.uint64),
                                         np.ascontiguousarray(hn, np.uint64), nonedge_weight, mu,
                                         C.byref(s), C.byref(steps))
        if rc:
            raise RuntimeError(self.error())
        return s.value, steps.value

    def random_relabel(self, n, seed):
        fwd = np.empty(n, np.uint32)
        self.lib.ref_random_relabel(n, seed, fwd)
        return fwd

    def init_embedding(self, n, dim, seed):
        out = np.empty((n, dim), np.float32)
        self.lib.ref_init_embedding(n, dim, seed, out)
        return out

    def load_edge_list(self, text: bytes):
        """load_edge_list: dict(rc, n, src, dst, labels, line, error)."""
        n, m, line = C.c_uint32(), C.c_uint64(), C.c_uint64()
        rc = self.lib.ref_load_edge_list(text, len(text), C.byref(n), C.byref(m), None, None, None, C.byref(line))
        if rc:
            return dict(rc=rc, line=line.value, error=self.error())
        src = np.zeros(m.value, np.uint32)
        dst = np.zeros(m.value, np.uint32)
        lab = np.zeros(n.value, np.uint64)
        self.lib.ref_load_edge_list(text, len(text), C.byref(n), C.byref(m), src.ctypes.data_as(C.c_void_p),
                                    dst.ctypes.data_as(C.c_void_p), lab.ctypes.data_as(C.c_void_p), C.byref(line))
        return dict(rc=0, n=n.value, src=src, dst=dst, labels=lab)

    def write_embedding_tsv(self, coords, labels=None, perm_forward=None) -> bytes:
        """write_embedding_tsv of the reference.  Runs in a numpy-free child process: inside a process that has
        imported numpy the reference's iostream/snprintf path segfaults in this image (the same call is fine from
        plain ctypes or C++), and this is test infrastructure, not something to debug in the reference."""
        import json
        import sys
        coords = np.ascontiguousarray(coords, np.float32)
        payload = json.dumps({"so": REF_SO, "n": int(coords.shape[0]), "dim": int(coords.shape[1]),
                              "bits": [int(v) for v in coords.view(np.uint32).ravel()],
                              "labels": None if labels is None else [int(v) for v in labels],
                              "perm": None if perm_forward is None else [int(v) for v in perm_forward]})
        child = (
            "import ctypes as C, json, sys\n"
            "p = json.loads(sys.stdin.read())\n"
            "L = C.CDLL(p['so'])\n"
            "L.ref_write_embedding_tsv.restype = C.c_long\n"
            "L.ref_write_embedding_tsv.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long]\n"
            "x = (C.c_uint32 * len(p['bits']))(*p['bits'])\n"
            "lab = (C.c_uint64 * p['n'])(*p['labels']) if p['labels'] is not None else None\n"
            "perm = (C.c_uint32 * p['n'])(*p['perm']) if p['perm'] is not None else None\n"
            "buf = C.create_string_buffer(1 << 22)\n"
            "k = L.ref_write_embedding_tsv(p['n'], p['dim'], C.cast(x, C.c_void_p), C.cast(lab, C.c_void_p) if lab else None,"
            " C.cast(perm, C.c_void_p) if perm else None, C.cast(buf, C.c_void_p), len(buf))\n"
            "sys.stdout.buffer.write(buf.raw[:k] if k >= 0 else b'')\n"
            "sys.exit(0 if k >= 0 else 1)\n")
        out = subprocess.run([sys.executable, "-c", child], input=payload.encode(), capture_output=True)
        if out.returncode != 0:
            raise RuntimeError("reference write_embedding_tsv failed: " + out.stderr.decode(errors="replace")[-300:])
        return out.stdout

    def save_graph_snapshot(self, n, src, dst) -> bytes:
        buf = C.create_string_buffer(16 + 8 * len(src) + 16)
        k = self.lib.ref_save_graph_snapshot(n, len(src), np.ascontiguousarray(src, np.uint32),
                                             np.ascontiguousarray(dst, np.uint32), C.cast(buf, C.c_void_p), len(buf))
        return buf.raw[:k]

    def pe_exact(self, n, src, dst, coords):
        pe = C.c_double()
        coords = np.ascontiguousarray(coords, np.float32)
        rc = self.lib.ref_pe_exact(n, len(src), np.ascontiguousarray(src, np.uint32),
                                   np.ascontiguousarray(dst, np.uint32), coords.shape[1], coords,
                                   C.byref(pe))
        if rc:
            raise RuntimeError(self.error())
        return pe.value


    def pe_sampled(self, n, src, dst, coords, samples_per_edge, seed):
        pe = C.c_double()
        coords = np.ascontiguousarray(coords, np.float32)
        rc = self.lib.ref_pe_sampled(n, len(src), np.ascontiguousarray(src, np.uint32),
                                     np.ascontiguousarray(dst, np.uint32), coords.shape[1], coords,
                                     samples_per_edge, seed, C.byref(pe))
        if rc:
            raise RuntimeError(self.error())
        return pe.value


class RefHash:
    def __init__(self, ref: Ref, n, src, dst, bits_override=0):
        self.ref, self.n = ref, n
        self.h = ref.lib.ref_hash_build(n, len(src), np.ascontiguousarray(src, np.uint32),
                                        np.ascontiguousarray(dst, np.uint32), bits_override)
        if not self.h:
            raise RuntimeError(ref.error())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_hash_free(self.h)
            self.h = None

    @property
    def size(self):
        return self.ref.lib.ref_hash_size(self.h)

    def probe(self, i, j):
        i = np.ascontiguousarray(i, np.uint32)
        j = np.ascontiguousarray(j, np.uint32)
        out = np.zeros(len(i), np.uint8)
        self.ref.lib.ref_hash_probe(self.h, i, j, len(i), out)
        return out

    def sample(self, anchors, states):
        anchors = np.ascontiguousarray(anchors, np.uint32)
        states = np.array(states, np.uint32)
        out = np.zeros(len(anchors), np.uint32)
        draws = C.c_uint64()
        rc = self.ref.lib.ref_sample_non_edges(self.h, self.n, anchors, states, len(anchors), out,
                                               C.byref(draws))
        return rc, out, states, draws.value


class RefEngine:
    """entropy_embed::EmbeddingEngine (engine.hpp:112-134) through the shim."""

    def __init__(self, ref: Ref, n, src, dst, dim, seed, lane_width=16, workers=1, fast_math=True,
                 hash_bits=0, relabel_period=0, max_iters=100, convergence_tol=1e-4,
                 convergence_window=5):
        self.ref, self.n, self.dim, self.m = ref, n, dim, len(src)
        self.h = ref.lib.ref_engine_create(n, len(src), np.ascontiguousarray(src, np.uint32),
                                           np.ascontiguousarray(dst, np.uint32), dim, lane_width,
                                           workers, int(fast_math), hash_bits, relabel_period,
                                           max_iters, convergence_tol, convergence_window, seed)
        if not self.h:
            raise RuntimeError(ref.error())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_engine_free(self.h)
            self.h = None

    @property
    def degenerate(self):
        return bool(self.ref.lib.ref_engine_degenerate(self.h))

    @property
    def sigma(self):
        return self.ref.lib.ref_engine_sigma(self.h)

    @property
    def hash_size(self):
        return self.ref.lib.ref_engine_hash_size(self.h)

    def work_graph(self):
        s = np.zeros(self.m, np.uint32)
        d = np.zeros(self.m, np.uint32)
        self.ref.lib.ref_engine_work_graph(self.h, s, d)
        return s, d

    def work_coords(self):
        out = np.zeros((self.n, self.dim), np.float32)
        self.ref.lib.ref_engine_work_coords(self.h, out)
        return out

    def probe(self, i, j):
        i = np.ascontiguousarray(i, np.uint32)
        j = np.ascontiguousarray(j, np.uint32)
        out = np.zeros(len(i), np.uint8)
        self.ref.lib.ref_engine_probe(self.h, i, j, len(i), out)
        return out

    def set_capture(self, on):
        self.ref.lib.ref_engine_set_capture(self.h, int(on))

    def iterate(self, capture=True):
        pe, sg = C.c_double(), C.c_double()
        y = z = None
        yp = zp = None
        if capture:
            y = np.zeros((self.n, self.dim), np.float64)
            z = np.zeros(self.n, np.float64)
            yp, zp = y.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p)
        rc = self.ref.lib.ref_engine_iterate(self.h, C.byref(pe), C.byref(sg), yp, zp)
        if rc:
            raise RuntimeError(f"rc={rc}: {self.ref.error()}")
        return dict(pe_estimate=pe.value, sigma=sg.value, y=y, z=z)

    def run(self, max_trace=100000):
        emb = np.zeros((self.n, self.dim), np.float32)
        trace = np.zeros(max_trace, np.float64)
        it, conv, deg = C.c_int(), C.c_int(), C.c_int()
        fs, nw = C.c_double(), C.c_double(1.0)
        fwd = np.zeros(self.n, np.uint32)
        he = np.zeros(BINS, np.uint64)
        hn = np.zeros(BINS, np.uint64)
        rc = self.ref.lib.ref_engine_run(self.h, emb.ctypes.data_as(C.c_void_p),
                                         trace.ctypes.data_as(C.c_void_p), max_trace, C.byref(it),
                                         C.byref(conv), C.byref(deg), C.byref(fs),
                                         fwd.ctypes.data_as(C.c_void_p),
                                         he.ctypes.data_as(C.c_void_p),
                                         hn.ctypes.data_as(C.c_void_p), C.byref(nw))
        if rc:
            raise RuntimeError(f"rc={rc}: {self.ref.error()}")
        return dict(embedding=emb, pe_trace=trace[:it.value].copy(), iterations=it.value,
                    converged=bool(conv.value), degenerate=bool(deg.value), final_sigma=fs.value,
                    relabel_forward=fwd, hist_edge=he, hist_nonedge=hn, nonedge_weight=nw.value)
