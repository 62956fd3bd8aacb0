"""Host-side mirror of the reference's engine interface over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/entropy_embed/engine.hpp
(``Graph``, ``IterationConfig``, ``EmbeddingEngine``, ``embed``) and errors.hpp; everything numerical happens
in libgempe_b200.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from ._capi import (HIST_BINS, INIT_NORMAL, INIT_REFERENCE, INIT_UNIFORM_PM1, MATH_EXACT, MATH_TABLES,
                    NEG_PER_EDGE_2, NEG_PER_VERTEX_K, RNG_PHILOX, RNG_REFERENCE)


# ---- errors.hpp:10-47 --------------------------------------------------------------------------------
class ConfigError(RuntimeError):
    """config_error: invalid configuration or request (exit code 1)."""


class DataError(RuntimeError):
    """data_error: structurally invalid data (exit code 2)."""


class NearCompleteGraphError(DataError):
    """near_complete_graph_error: a sample stream hit the 10^4 retry cap."""


class DivergenceError(RuntimeError):
    """divergence_error: a coordinate became non-finite (exit code 3)."""


class CudaError(RuntimeError):
    """CUDA runtime failure or no device: the path has no CPU fallback."""


def _raise(rc: int, msg: str):
    if rc == _capi.OK:
        return
    if rc == _capi.ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _capi.ERR_DIVERGENCE:
        raise DivergenceError(msg)
    if rc == _capi.ERR_CUDA:
        raise CudaError(msg)
    if "near-complete" in msg:
        raise NearCompleteGraphError(msg)
    raise DataError(msg)


@dataclass
class Graph:
    """graph.hpp:12-23: canonical undirected graph, ids 0..n-1, SoA edge arrays."""
    n: int
    src: np.ndarray
    dst: np.ndarray

    def __post_init__(self):
        self.src = np.ascontiguousarray(self.src, np.uint32)
        self.dst = np.ascontiguousarray(self.dst, np.uint32)
        if self.src.shape != self.dst.shape:
            raise DataError("src/dst length mismatch")

    def edge_count(self) -> int:
        return int(self.src.size)

    def pair_count(self) -> int:
        return self.n * (self.n - 1) // 2 if self.n > 0 else 0


@dataclass
class IterationConfig:
    """engine.hpp:29-38 plus the BASELINE extensions (negatives per vertex, device)."""
    max_iters: int = 100
    lane_width: int = 16
    workers: int = 0
    convergence_tol: float = 1e-4
    convergence_window: int = 5
    relabel_period: int = 0
    fast_math: bool = True
    hash_bits: Optional[int] = None
    neg_mode: int = NEG_PER_EDGE_2
    negatives: int = 0
    device: int = 0
    host_sigma: bool = False  # True: sigma search on the host instead of the device kernel
    deterministic: bool = False  # True: sorted sample buckets, byte-identical results run to run
    batch_rounds: int = 0  # run(): whole iterations queued per host round trip (0 auto, 1 every round, < 0 host loop)
    devices: Optional[list] = None  # several GPUs of this process: vertices sharded over them (gempe_engine_create_multi)


@dataclass
class IterationStats:
    pe_estimate: float = 0.0
    sigma: float = 0.0


@dataclass
class EmbedResult:
    """engine.hpp:98-107."""
    embedding: np.ndarray
    pe_trace: np.ndarray
    final_sigma: float = 1.0
    converged: bool = False
    degenerate: bool = False
    iterations: int = 0
    relabel_forward: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    last_hist_edge: np.ndarray = field(default_factory=lambda: np.zeros(HIST_BINS, np.uint64))
    last_hist_nonedge: np.ndarray = field(default_factory=lambda: np.zeros(HIST_BINS, np.uint64))
    last_nonedge_weight: float = 1.0


class Context:
    """One GPU shard of the engine (gempe_ctx): the Jacobi round and its test hooks."""

    def __init__(self, g: Graph, dim: int, seed: int = 1, *, neg_mode=NEG_PER_EDGE_2, negatives=0,
                 math=MATH_TABLES, rng=RNG_REFERENCE, hash_bits=0, relabel=True, device=0, rank=0, world=1,
                 comm_chunks=1, chunk_entries=0, deterministic=False, precise_distance=False, kernel_variant=0, bucket_mode=0,
                 exchange=False):
        self._L = _capi.load()
        self._h = C.c_void_p()
        opt = _capi.Options()
        self._L.gempe_default_options(C.byref(opt))
        opt.dim, opt.seed, opt.neg_mode, opt.negatives = dim, seed, neg_mode, negatives
        opt.math, opt.rng, opt.hash_bits, opt.relabel = math, rng, hash_bits or 0, int(relabel)
        opt.device, opt.rank, opt.world, opt.comm_chunks = device, rank, world, comm_chunks
        opt.chunk_entries, opt.deterministic = chunk_entries, int(deterministic)
        opt.precise_distance, opt.kernel_variant = int(precise_distance), kernel_variant
        opt.bucket_mode = bucket_mode
        opt.exchange = int(exchange)  # 0 off, 1 on, 2 on with the exchange left to the caller even for one rank
        self.n, self.m, self.dim = int(g.n), g.edge_count(), int(dim)
        rc = self._L.gempe_create(C.byref(self._h), g.n, self.m, _capi.ptr(g.src), _capi.ptr(g.dst), C.byref(opt))
        if rc != _capi.OK:
            self._h = C.c_void_p()
            _raise(rc, self._L.gempe_last_error(None).decode())

    # -- lifetime ------------------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._L.gempe_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != _capi.OK:
            _raise(rc, self._L.gempe_last_error(self._h).decode())

    # -- properties ----------------------------------------------------------------------------------
    @property
    def degenerate(self) -> bool:
        return bool(self._L.gempe_is_degenerate(self._h))

    @property
    def hash_bits(self) -> int:
        return self._L.gempe_hash_bits(self._h)

    @property
    def sample_slots(self) -> int:
        return self._L.gempe_sample_slots(self._h)

    @property
    def pair_terms(self) -> int:
        return self._L.gempe_pair_terms(self._h)

    @property
    def algorithmic_bytes(self) -> int:
        return self._L.gempe_algorithmic_bytes(self._h)

    @property
    def kernel_launches(self) -> int:
        return self._L.gempe_kernel_launches(self._h)

    @property
    def bucket_spills(self) -> int:
        return self._L.gempe_bucket_spills(self._h)

    @property
    def row_stride(self) -> int:
        return self._L.gempe_row_stride(self._h)

    @property
    def padded_rows(self) -> int:
        return self._L.gempe_padded_rows(self._h)

    @property
    def block_rows(self) -> int:
        return self._L.gempe_block_rows(self._h)

    # -- graph / coordinates -------------------------------------------------------------------------
    def work_graph(self):
        src = np.zeros(self.m, np.uint32)
        dst = np.zeros(self.m, np.uint32)
        to_work = np.zeros(self.n, np.uint32)
        self._check(self._L.gempe_get_work_graph(self._h, _capi.ptr(src), _capi.ptr(dst), _capi.ptr(to_work)))
        return src, dst, to_work

    def set_coords(self, x_work: np.ndarray):
        x = np.ascontiguousarray(x_work, np.float32)
        if x.shape != (self.n, self.dim):
            raise ConfigError(f"coordinates must be {self.n}x{self.dim}")
        self._check(self._L.gempe_set_coords(self._h, _capi.ptr(x)))

    def get_coords(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.n, self.dim), np.float32)
        self._check(self._L.gempe_get_coords(self._h, _capi.ptr(out)))
        return out

    def init_coords(self, rule=INIT_REFERENCE, seed=1, std=0.01):
        self._check(self._L.gempe_init_coords(self._h, rule, seed, std))

    def relabel(self, relabel_seed: int):
        self._check(self._L.gempe_relabel(self._h, relabel_seed))

    # -- the round -----------------------------------------------------------------------------------
    def iterate(self, mu: float, sigma: float, iter_index: int):
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        self._check(self._L.gempe_iterate(self._h, mu, sigma, iter_index, _capi.ptr(he), _capi.ptr(hn)))
        return he, hn

    def step_host(self, x_in: np.ndarray, x_out: np.ndarray, mu: float, sigma: float, iter_index: int):
        """The round on host buffers (X_t in, X_{t+1} out), copies overlapped with the kernels."""
        if x_in.dtype != np.float32 or x_out.dtype != np.float32 or x_in.shape != (self.n, self.dim) \
                or x_out.shape != (self.n, self.dim) or not x_in.flags.c_contiguous or not x_out.flags.c_contiguous:
            raise ConfigError(f"coordinates must be C-contiguous float32 {self.n}x{self.dim}")
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        self._check(self._L.gempe_step_host(self._h, _capi.ptr(x_in), _capi.ptr(x_out), mu, sigma, iter_index,
                                            _capi.ptr(he), _capi.ptr(hn)))
        return he, hn

    def iterate_async(self, mu: float, sigma: float, iter_index: int):
        self._check(self._L.gempe_iterate_async(self._h, mu, sigma, iter_index))

    def sync(self):
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        self._check(self._L.gempe_sync(self._h, _capi.ptr(he), _capi.ptr(hn)))
        return he, hn

    # -- device-resident sigma feedback ----------------------------------------------------------------
    def set_sigma(self, mu: float, sigma: float):
        self._check(self._L.gempe_set_sigma(self._h, mu, sigma))

    def iterate_auto(self, iter_index: int):
        """One round with the device's sigma, then the device sigma search.  Returns (sigma, pe, nonedge_weight,
        hist_edge, hist_nonedge)."""
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        s, pe, nw = C.c_double(), C.c_double(), C.c_double()
        self._check(self._L.gempe_iterate_auto(self._h, iter_index, C.byref(s), C.byref(pe), C.byref(nw), _capi.ptr(he),
                                               _capi.ptr(hn)))
        return s.value, pe.value, nw.value, he, hn

    def pe_sampled(self, samples_per_edge: int = 2, seed: int = 1) -> dict:
        """metrics.cpp pe_sampled of the current coordinates, on the device: dict(pe, mu_star, sigma_star, h_basic,
        compression_ratio, grid_pe, nonedge_samples)."""
        rep = _capi.PeReportC()
        self._check(self._L.gempe_pe_sampled(self._h, samples_per_edge, seed, C.byref(rep)))
        return {name: getattr(rep, name) for name, _ in rep._fields_}

    # -- runs queued without host round trips ----------------------------------------------------------
    def run_begin(self, mu: float, sigma: float, first_iter: int = 0, window: int = 5, tol: float = 1e-4,
                  max_rounds: int = 100):
        self._run_cap = int(max_rounds)
        self._check(self._L.gempe_run_begin(self._h, mu, sigma, first_iter, window, tol, max_rounds))

    def run_enqueue(self, rounds: int, stop_at: int, use_graph: bool = True):
        self._check(self._L.gempe_run_enqueue(self._h, rounds, stop_at, int(use_graph)))

    def run_poll(self) -> dict:
        """Waits for the queued rounds; dict(rounds_done, converged, failed, improved_at, best_pe, sigma, pe_estimate,
        last_nonedge_weight, draws, pe_trace, sigma_trace, hist_edge, hist_nonedge)."""
        st = _capi.RunStatusC()
        pe = np.zeros(self._run_cap, np.float64)
        sg = np.zeros(self._run_cap, np.float64)
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        self._check(self._L.gempe_run_poll(self._h, C.byref(st), _capi.ptr(pe), _capi.ptr(sg), self._run_cap, _capi.ptr(he),
                                           _capi.ptr(hn)))
        out = {name: getattr(st, name) for name, _ in st._fields_}
        k = min(int(st.rounds_done), self._run_cap)
        out.update(pe_trace=pe[:k], sigma_trace=sg[:k], hist_edge=he, hist_nonedge=hn)
        return out

    def graph_capture(self, mu: float, sigma: float, first_iter: int, count: int):
        """Captures `count` rounds into a CUDA graph (replayed by graph_launch)."""
        self._check(self._L.gempe_graph_capture(self._h, mu, sigma, first_iter, count))

    def graph_launch(self):
        self._check(self._L.gempe_graph_launch(self._h))

    def iterate_auto_async(self, iter_index: int):
        self._check(self._L.gempe_iterate_auto_async(self._h, iter_index))

    def sigma_state(self):
        s, pe, nw = C.c_double(), C.c_double(), C.c_double()
        self._check(self._L.gempe_get_sigma_state(self._h, C.byref(s), C.byref(pe), C.byref(nw)))
        return s.value, pe.value, nw.value

    def sigma_update_async(self):
        self._check(self._L.gempe_sigma_update_async(self._h))

    def device_tallies(self) -> int:
        return self._L.gempe_device_tallies(self._h)

    def elapsed_ms(self):
        out = (C.c_float * 3)()
        self._check(self._L.gempe_elapsed_ms(self._h, C.byref(out)))
        return float(out[0]), float(out[1]), float(out[2])

    def set_capture(self, on: bool):
        self._check(self._L.gempe_set_capture(self._h, int(on)))

    def get_yz(self):
        y = np.zeros((self.n, self.dim), np.float64)
        z = np.zeros(self.n, np.float64)
        self._check(self._L.gempe_get_yz(self._h, _capi.ptr(y), _capi.ptr(z)))
        return y, z

    def get_yz_rows(self, rows):
        rows = np.ascontiguousarray(rows, np.uint32)
        y = np.zeros((rows.size, self.dim), np.float64)
        z = np.zeros(rows.size, np.float64)
        self._check(self._L.gempe_get_yz_rows(self._h, _capi.ptr(rows), rows.size, _capi.ptr(y), _capi.ptr(z)))
        return y, z

    def get_coords_rows(self, rows):
        rows = np.ascontiguousarray(rows, np.uint32)
        x = np.zeros((rows.size, self.dim), np.float32)
        self._check(self._L.gempe_get_coords_rows(self._h, _capi.ptr(rows), rows.size, _capi.ptr(x)))
        return x

    # -- bit-exact hooks -----------------------------------------------------------------------------
    def probe(self, i, j) -> np.ndarray:
        i = np.ascontiguousarray(i, np.uint32)
        j = np.ascontiguousarray(j, np.uint32)
        out = np.zeros(i.size, np.uint8)
        self._check(self._L.gempe_probe(self._h, _capi.ptr(i), _capi.ptr(j), i.size, _capi.ptr(out)))
        return out

    def sample(self, iter_index: int):
        partners = np.zeros(max(self.sample_slots, 1), np.uint32)
        draws = C.c_uint64()
        self._check(self._L.gempe_sample(self._h, iter_index, _capi.ptr(partners), C.byref(draws)))
        return partners[:self.sample_slots], draws.value

    # -- sharded stepping ----------------------------------------------------------------------------
    def set_stream(self, cuda_stream: int):
        self._check(self._L.gempe_set_stream(self._h, C.c_void_p(cuda_stream)))

    def device_coords(self, which: int) -> int:
        return self._L.gempe_device_coords(self._h, which)

    def begin_round(self, mu, sigma, iter_index):
        self._check(self._L.gempe_begin_round(self._h, mu, sigma, iter_index))

    def begin_round_auto(self, iter_index):
        self._check(self._L.gempe_begin_round_auto(self._h, iter_index))

    def exchange_layout(self):
        """(send_records, recv_records, send_counts, recv_counts) device addresses and the per-region capacity."""
        ptrs = [C.c_void_p() for _ in range(4)]
        cap = C.c_uint32()
        self._check(self._L.gempe_exchange_layout(self._h, *[C.byref(p) for p in ptrs], C.byref(cap)))
        return tuple(p.value for p in ptrs) + (cap.value,)

    def bucket_received(self):
        self._check(self._L.gempe_bucket_received(self._h))

    # fused update + broadcast over peer memory
    def coords_ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(128)
        self._check(self._L.gempe_coords_ipc_handles(self._h, buf))
        return buf.raw

    def open_peer(self, handles: bytes):
        self._check(self._L.gempe_open_peer(self._h, C.c_char_p(handles)))

    def add_peer_pointers(self, x_parity0: int, x_parity1: int):
        self._check(self._L.gempe_add_peer_pointers(self._h, C.c_void_p(x_parity0), C.c_void_p(x_parity1)))

    # direct sample exchange
    def exchange_ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        self._check(self._L.gempe_exchange_ipc_handle(self._h, buf))
        return buf.raw

    def open_peer_exchange(self, peer_rank: int, handle: bytes):
        self._check(self._L.gempe_open_peer_exchange(self._h, peer_rank, C.c_char_p(handle)))

    def add_peer_exchange_pointer(self, peer_rank: int, recv_area: int):
        self._check(self._L.gempe_add_peer_exchange_pointer(self._h, peer_rank, C.c_void_p(recv_area)))

    @property
    def exchange_recv_area(self) -> int:
        return self._L.gempe_exchange_recv_area(self._h)

    def clear_peers(self):
        self._check(self._L.gempe_clear_peers(self._h))

    def device_coords_parity(self, parity: int) -> int:
        return self._L.gempe_device_coords_parity(self._h, parity)

    @property
    def coords_parity(self) -> int:
        return self._L.gempe_coords_parity(self._h)

    def gather_chunk(self, chunk: int):
        self._check(self._L.gempe_gather_chunk(self._h, chunk))

    def end_round(self):
        self._check(self._L.gempe_end_round(self._h))


class Group:
    """Several GPUs in one process (gempe_group): one context per listed device, vertices sharded over them.  A device
    may be listed more than once (several ranks on one GPU: what the tests use)."""

    GROUP_COPY_ENGINES = 1

    def __init__(self, g: Graph, dim: int, seed: int = 1, *, devices=(0,), copy_engines=False, neg_mode=NEG_PER_EDGE_2,
                 negatives=0, math=MATH_TABLES, rng=RNG_REFERENCE, hash_bits=0, relabel=True, chunk_entries=0,
                 deterministic=False, precise_distance=False, bucket_mode=0):
        self._L = _capi.load()
        self._h = C.c_void_p()
        opt = _capi.Options()
        self._L.gempe_default_options(C.byref(opt))
        opt.dim, opt.seed, opt.neg_mode, opt.negatives = dim, seed, neg_mode, negatives
        opt.math, opt.rng, opt.hash_bits, opt.relabel = math, rng, hash_bits or 0, int(relabel)
        opt.chunk_entries, opt.deterministic = chunk_entries, int(deterministic)
        opt.precise_distance, opt.bucket_mode = int(precise_distance), bucket_mode
        self.n, self.m, self.dim = int(g.n), g.edge_count(), int(dim)
        dev = (C.c_int * len(devices))(*[int(d) for d in devices])
        rc = self._L.gempe_group_create(C.byref(self._h), g.n, self.m, _capi.ptr(g.src), _capi.ptr(g.dst), C.byref(opt),
                                        C.cast(dev, C.c_void_p), len(devices),
                                        self.GROUP_COPY_ENGINES if copy_engines else 0)
        if rc != _capi.OK:
            self._h = C.c_void_p()
            _raise(rc, self._L.gempe_group_last_error(None).decode())

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._L.gempe_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != _capi.OK:
            _raise(rc, self._L.gempe_group_last_error(self._h).decode())

    @property
    def world(self) -> int:
        return self._L.gempe_group_world(self._h)

    @property
    def exchange_path(self) -> str:
        return self._L.gempe_group_exchange_path(self._h).decode()

    def set_coords(self, x_work: np.ndarray):
        x = np.ascontiguousarray(x_work, np.float32)
        if x.shape != (self.n, self.dim):
            raise ConfigError(f"coordinates must be {self.n}x{self.dim}")
        self._check(self._L.gempe_group_set_coords(self._h, _capi.ptr(x)))

    def init_coords(self, rule=INIT_REFERENCE, seed=1, std=0.01):
        self._check(self._L.gempe_group_init_coords(self._h, rule, seed, std))

    def get_coords(self) -> np.ndarray:
        out = np.empty((self.n, self.dim), np.float32)
        self._check(self._L.gempe_group_get_coords(self._h, _capi.ptr(out)))
        return out

    def iterate(self, mu: float, sigma: float, iter_index: int):
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        self._check(self._L.gempe_group_iterate(self._h, mu, sigma, iter_index, _capi.ptr(he), _capi.ptr(hn)))
        return he, hn

    def set_sigma(self, mu: float, sigma: float):
        self._check(self._L.gempe_group_set_sigma(self._h, mu, sigma))

    def iterate_auto(self, iter_index: int):
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        s, pe, nw = C.c_double(), C.c_double(), C.c_double()
        self._check(self._L.gempe_group_iterate_auto(self._h, iter_index, C.byref(s), C.byref(pe), C.byref(nw),
                                                     _capi.ptr(he), _capi.ptr(hn)))
        return s.value, pe.value, nw.value, he, hn

    def relabel(self, relabel_seed: int):
        self._check(self._L.gempe_group_relabel(self._h, relabel_seed))

    def replicas_agree(self) -> bool:
        rc = self._L.gempe_group_replicas_agree(self._h)
        if rc < 0:
            _raise(-rc, self._L.gempe_group_last_error(self._h).decode())
        return rc == 1


class EmbeddingEngine:
    """engine.hpp:112-134 (run-level facade, gempe_engine)."""

    def __init__(self, g: Graph, dim: int, cfg: IterationConfig, seed: int):
        self._L = _capi.load()
        self._h = C.c_void_p()
        c = _capi.IterationConfigC()
        self._L.gempe_default_iteration_config(C.byref(c))
        c.max_iters, c.lane_width, c.workers = cfg.max_iters, cfg.lane_width, cfg.workers
        c.convergence_tol, c.convergence_window = cfg.convergence_tol, cfg.convergence_window
        c.relabel_period, c.fast_math = cfg.relabel_period, int(cfg.fast_math)
        c.hash_bits = 0 if cfg.hash_bits is None else cfg.hash_bits
        if cfg.hash_bits is not None and not (1 <= cfg.hash_bits <= 31):
            raise ConfigError("hash table bits must be in [1,31]")
        c.neg_mode, c.negatives, c.device = cfg.neg_mode, cfg.negatives, cfg.device
        c.host_sigma = int(cfg.host_sigma)
        c.deterministic = int(cfg.deterministic)
        c.batch_rounds = int(cfg.batch_rounds)
        self.n, self.m, self.dim = int(g.n), g.edge_count(), int(dim)
        self._pe_trace = []
        devices = list(cfg.devices) if cfg.devices else []
        dev = (C.c_int * max(1, len(devices)))(*devices)
        rc = self._L.gempe_engine_create_multi(C.byref(self._h), g.n, self.m, _capi.ptr(g.src), _capi.ptr(g.dst), dim,
                                               C.byref(c), seed, C.cast(dev, C.c_void_p) if devices else None,
                                               len(devices))
        if rc != _capi.OK:
            self._h = C.c_void_p()
            _raise(rc, self._L.gempe_last_error(None).decode())

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._L.gempe_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != _capi.OK:
            _raise(rc, self._L.gempe_engine_last_error(self._h).decode())

    def context(self) -> "Context":
        """Borrowed low-level view (work graph, coordinates, hooks) of the engine's device context."""
        ctx = Context.__new__(Context)
        ctx._L = self._L
        ctx._h = C.c_void_p(self._L.gempe_engine_context(self._h))
        ctx.n, ctx.m, ctx.dim = self.n, self.m, self.dim
        ctx.close = lambda: None  # borrowed: never destroys
        return ctx

    def degenerate(self) -> bool:
        return bool(self._L.gempe_engine_degenerate(self._h))

    def iteration(self) -> int:
        return self._L.gempe_engine_iteration(self._h)

    def sigma(self) -> float:
        return self._L.gempe_engine_sigma(self._h)

    def pe_trace(self):
        return list(self._pe_trace)

    def work_graph(self):
        return self.context().work_graph()

    def work_coords(self) -> np.ndarray:
        return self.context().get_coords()

    def run_single_iteration(self) -> IterationStats:
        pe, sg = C.c_double(), C.c_double()
        self._check(self._L.gempe_engine_run_single_iteration(self._h, C.byref(pe), C.byref(sg)))
        self._pe_trace.append(pe.value)
        return IterationStats(pe.value, sg.value)

    def run(self, max_trace: int = 1 << 20) -> EmbedResult:
        emb = np.zeros((self.n, self.dim), np.float32)
        trace = np.zeros(max_trace, np.float64)
        fwd = np.zeros(self.n, np.uint32)
        he = np.zeros(HIST_BINS, np.uint64)
        hn = np.zeros(HIST_BINS, np.uint64)
        r = _capi.EmbedResultC()
        r.embedding, r.pe_trace, r.pe_trace_cap = _capi.ptr(emb), _capi.ptr(trace), max_trace
        r.relabel_forward, r.last_hist_edge, r.last_hist_nonedge = _capi.ptr(fwd), _capi.ptr(he), _capi.ptr(hn)
        self._check(self._L.gempe_engine_run(self._h, C.byref(r)))
        self._pe_trace = list(trace[:r.pe_trace_len])
        return EmbedResult(emb, trace[:r.pe_trace_len].copy(), r.final_sigma, bool(r.converged),
                           bool(r.degenerate), r.iterations, fwd, he, hn, r.last_nonedge_weight)


def embed(g: Graph, dim: int, cfg: Optional[IterationConfig] = None, seed: int = 1, *, iterations=None,
          negatives=None) -> EmbedResult:
    """``embed(g, dim, cfg, seed)`` (engine.hpp:170-171).  The BASELINE convenience form
    ``embed(g, dim, iterations=I, negatives=k, seed=s)`` selects k draws per vertex."""
    cfg = cfg or IterationConfig()
    if iterations is not None:
        cfg.max_iters = iterations
    if negatives is not None:
        cfg.neg_mode, cfg.negatives = NEG_PER_VERTEX_K, negatives
    engine = EmbeddingEngine(g, dim, cfg, seed)
    try:
        return engine.run()
    finally:
        engine.close()


def trim_device_cache():
    """Returns the device memory cached from destroyed contexts / engines to the driver (gempe_trim_device_cache)."""
    _capi.load().gempe_trim_device_cache()


def alloc_host(shape, dtype=np.float32) -> np.ndarray:
    """A numpy array on page-locked host memory (gempe_alloc_host): step_host / set_coords / get_coords on it run at the
    PCIe rate.  Release it with free_host(array) -- not by dropping the last reference."""
    L = _capi.load()
    dt = np.dtype(dtype)
    count = int(np.prod(shape))
    p = L.gempe_alloc_host(max(1, count * dt.itemsize))
    if not p:
        raise CudaError((L.gempe_last_error(None) or b"").decode())
    buf = (C.c_char * (count * dt.itemsize)).from_address(p)
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


def free_host(a: np.ndarray):
    _capi.load().gempe_free_host(C.c_void_p(a.ctypes.data))


# ---- host numerics (no GPU) ----------------------------------------------------------------------------
def fastmath_table(which: int):
    out = np.zeros(67, np.float64)
    odd = _capi.load().gempe_host_fastmath_table(which, out)
    if odd < 0:
        raise ConfigError("table build failed")
    return out, odd


def optimize_sigma(hist_edge, hist_nonedge, nonedge_weight, mu=1.5):
    steps = C.c_int()
    s = _capi.load().gempe_host_optimize_sigma(np.ascontiguousarray(hist_edge, np.uint64),
                                               np.ascontiguousarray(hist_nonedge, np.uint64), nonedge_weight, mu,
                                               C.byref(steps))
    if s != s:
        raise ConfigError("cannot optimize sigma on an empty histogram")
    return s, steps.value


def histogram_objective(hist_edge, hist_nonedge, nonedge_weight, mu, sigma):
    return _capi.load().gempe_host_histogram_objective(np.ascontiguousarray(hist_edge, np.uint64),
                                                      np.ascontiguousarray(hist_nonedge, np.uint64),
                                                      nonedge_weight, mu, sigma)


def histogram_objective_dsigma(hist_edge, hist_nonedge, nonedge_weight, mu, sigma):
    return _capi.load().gempe_host_histogram_objective_dsigma(np.ascontiguousarray(hist_edge, np.uint64),
                                                             np.ascontiguousarray(hist_nonedge, np.uint64),
                                                             nonedge_weight, mu, sigma)


def random_relabel(n: int, seed: int) -> np.ndarray:
    fwd = np.zeros(n, np.uint32)
    _capi.load().gempe_host_random_relabel(n, seed, fwd)
    return fwd


def mix_seed(seed: int, component: int) -> int:
    return _capi.load().gempe_host_mix_seed(seed, component)


# ---- graph ingest / embedding export (host side) -------------------------------------------------------
class ParseError(DataError):
    """parse_error: malformed input text; `line` is the 1-based offending line (errors.hpp:10-19)."""

    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


def _take_graph(L, gc):
    try:
        src = np.ctypeslib.as_array(gc.src, (gc.m,)).copy()
        dst = np.ctypeslib.as_array(gc.dst, (gc.m,)).copy()
        labels = np.ctypeslib.as_array(gc.raw_labels, (gc.n,)).copy() if gc.raw_labels else None
        return Graph(gc.n, src, dst), labels
    finally:
        L.gempe_graph_free(C.byref(gc))


def _raise_io(L, rc, line):
    msg = L.gempe_last_error(None).decode(errors="replace")
    if rc == _capi.ERR_DATA and line:
        raise ParseError(msg, line)
    _raise(rc, msg)


def load_edge_list(text) -> tuple:
    """load_edge_list (graph.cpp:75-133).  Returns (Graph, raw_labels)."""
    L = _capi.load()
    data = text.encode() if isinstance(text, str) else bytes(text)
    gc, line = _capi.GraphC(), C.c_uint64()
    rc = L.gempe_parse_edge_list(data, len(data), C.byref(gc), C.byref(line))
    if rc != _capi.OK:
        _raise_io(L, rc, line.value)
    return _take_graph(L, gc)


def load_graph_snapshot(data: bytes) -> Graph:
    L = _capi.load()
    gc = _capi.GraphC()
    rc = L.gempe_parse_graph_snapshot(bytes(data), len(data), C.byref(gc))
    if rc != _capi.OK:
        _raise_io(L, rc, 0)
    return _take_graph(L, gc)[0]


def load_graph_file(path: str) -> tuple:
    L = _capi.load()
    gc, line = _capi.GraphC(), C.c_uint64()
    rc = L.gempe_load_graph_file(path.encode(), C.byref(gc), C.byref(line))
    if rc != _capi.OK:
        _raise_io(L, rc, line.value)
    return _take_graph(L, gc)


def save_graph_snapshot(path: str, g: Graph):
    L = _capi.load()
    rc = L.gempe_write_graph_snapshot(path.encode(), g.n, g.edge_count(), _capi.ptr(g.src), _capi.ptr(g.dst))
    if rc != _capi.OK:
        _raise_io(L, rc, 0)


def write_embedding_tsv(path: str, coords: np.ndarray, labels=None, perm_forward=None):
    """write_embedding_tsv (io.cpp:17-46)."""
    L = _capi.load()
    x = np.ascontiguousarray(coords, np.float32)
    lab = None if labels is None else np.ascontiguousarray(labels, np.uint64)
    perm = None if perm_forward is None else np.ascontiguousarray(perm_forward, np.uint32)
    if lab is not None and lab.size != x.shape[0]:
        raise DataError("label count does not match embedding rows")
    rc = L.gempe_write_embedding_tsv(path.encode(), x.shape[0], x.shape[1], _capi.ptr(x), _capi.ptr(lab), _capi.ptr(perm))
    if rc != _capi.OK:
        _raise_io(L, rc, 0)
