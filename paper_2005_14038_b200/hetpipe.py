"""Thin ctypes binding of libhetpipe (include/hetpipe.h): argument marshalling
only -- every step of the WSP path runs in the library's C++ controller and
sm_100a kernels. There is no CPU fallback: if the library is missing or no
CUDA device is usable, these calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HP_LIB: another build of the same library (e.g. a tuning variant) -- still
# the in-tree CUDA library; there is no CPU fallback
LIB_PATH = os.environ.get("HP_LIB") or os.path.join(_HERE, "libhetpipe.so")

HP_OK, HP_WOULD_BLOCK = 0, 1
HP_ERR_INVALID, HP_ERR_PROTOCOL, HP_ERR_CUDA = -1, -2, -3
HP_ERR_COMM, HP_ERR_OOM, HP_ERR_STATE = -4, -5, -6
STATUS_NAMES = {0: "HP_OK", 1: "HP_WOULD_BLOCK", -1: "HP_ERR_INVALID",
                -2: "HP_ERR_PROTOCOL", -3: "HP_ERR_CUDA", -4: "HP_ERR_COMM",
                -5: "HP_ERR_OOM", -6: "HP_ERR_STATE"}


class hp_config(C.Structure):
    _fields_ = [("num_vw", C.c_int32), ("Nm", C.c_int32), ("D", C.c_int32),
                ("waves", C.c_int32), ("nparams", C.c_int64),
                ("param_begin", C.c_int64), ("param_count", C.c_int64),
                ("lr", C.c_float), ("momentum", C.c_float), ("seed", C.c_uint64),
                ("grad_mode", C.c_int32), ("w0_mode", C.c_int32),
                ("pull_policy", C.c_int32), ("local_semantics", C.c_int32),
                ("apply_mode", C.c_int32), ("acc_slots", C.c_int32),
                ("merge_ticks", C.c_int32), ("world", C.c_int32), ("rank", C.c_int32),
                ("vw_span", C.c_int32), ("device", C.c_int32), ("stream", C.c_void_p),
                ("transport", C.c_int32), ("reserved", C.c_int32),
                ("update_freq", C.c_int32), ("lr_schedule", C.c_int32),
                ("conv_a", C.c_float), ("conv_sigma", C.c_float), ("ps_bounds", C.c_void_p),
                ("arena", C.c_void_p)]

XPORT_PEER, XPORT_NCCL, XPORT_NVLS = 0, 1, 2
XPORTS = {"peer": XPORT_PEER, "nccl": XPORT_NCCL, "nvls": XPORT_NVLS}


class hp_stats(C.Structure):
    _fields_ = [("commits", C.c_int64), ("applied", C.c_int64),
                ("launches", C.c_int64), ("ticks", C.c_int64),
                ("alg_bytes", C.c_double), ("wait_ticks", C.c_int64 * 8),
                ("pulls", C.c_int64 * 8), ("nvl_bytes", C.c_double),
                ("lockstep_batches", C.c_int64), ("apply_batches", C.c_int64),
                ("desc_splits", C.c_int64)]


class hp_unit(C.Structure):
    _fields_ = [("params", C.c_int64), ("fwd_flops", C.c_int64), ("act_out", C.c_int64),
                ("act_resident", C.c_int64)]


class hp_gpu(C.Structure):
    _fields_ = [("flops_per_s", C.c_double), ("mem_bytes", C.c_double), ("node", C.c_int32),
                ("reserved", C.c_int32)]


class HetPipeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None

EXPORTS = {
    "hp_config_size": (C.c_size_t, []),
    "hp_config_default": (None, [C.POINTER(hp_config)]),
    "hp_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int32,
                          C.c_int64, C.c_float]),
    "hp_init_ex": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(hp_config)]),
    "hp_accumulate_minibatch": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]),
    "hp_accumulate_minibatch_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]),
    "hp_push_wave": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "hp_clock": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "hp_pull": (C.c_int, [C.c_void_p, C.c_int32]),
    "hp_tick_end": (C.c_int, [C.c_void_p]),
    "hp_flush": (C.c_int, [C.c_void_p]),
    "hp_set_tick": (C.c_int, [C.c_void_p, C.c_int64]),
    "hp_comm_unique_id": (C.c_int, [C.c_void_p]),
    "hp_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hp_connect": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "hp_arena_bytes": (C.c_int64, [C.POINTER(hp_config)]),
    "hp_connect_symmetric": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hp_schedule_begin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "hp_schedule_advance": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "hp_run_schedule": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "hp_schedule_set_host_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "hp_schedule_capture": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_void_p)]),
    "hp_graph_launch": (C.c_int, [C.c_void_p]),
    "hp_graph_destroy": (None, [C.c_void_p]),
    "hp_launch_floor": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_float)]),
    "hp_drain": (C.c_int, [C.c_void_p]),
    "hp_sync": (C.c_int, [C.c_void_p]),
    "hp_read_weights": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]),
    "hp_trace_dump": (C.c_int, [C.c_void_p, C.c_char_p]),
    "hp_trace_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "hp_get_stats": (C.c_int, [C.c_void_p, C.POINTER(hp_stats)]),
    "hp_profile_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "hp_profile_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_int64)]),
    "hp_profile_launches": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(C.c_int64)]),
    "hp_profile_link": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_int64)]),
    "hp_profile_streams": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_int64)]),
    "hp_profile_sync_latency": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.POINTER(C.c_int64)]),
    "hp_partition": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                               C.c_int32, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
    "hp_max_m": (C.c_int32, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                             C.c_double, C.c_double]),
    "hp_pipeline_simulate": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                                       C.c_void_p]),
    "hp_pipeline_tau_latency": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "hp_s_global": (C.c_int64, [C.c_int32, C.c_int32]),
    "hp_s_global_f": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "hp_version_floor": (C.c_int64, [C.c_int64, C.c_int32, C.c_int32]),
    "hp_last_error": (C.c_char_p, [C.c_void_p]),
    "hp_version": (C.c_char_p, []),
    "hp_finalize": (None, [C.c_void_p]),
}


def _bind(lib: C.CDLL) -> C.CDLL:
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load() -> C.CDLL:
    """Load libhetpipe.so (built by paper_2005_14038_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2005_14038_b200.build`")
        lib = _bind(C.CDLL(LIB_PATH))
        if lib.hp_config_size() != C.sizeof(hp_config):
            raise ImportError("hp_config layout of the binding does not match libhetpipe.so")
        _lib = lib
    return _lib


def load_test_library(path: str) -> C.CDLL:
    """Bind another build of the same ABI (tests/emu's host-emulated engine,
    used only by CPU tests of the host logic). Never used by the product."""
    return _bind(C.CDLL(path))


def config_from(cfg, **overrides) -> hp_config:
    """hp_config from a workloads.WSPConfig (plus keyword overrides)."""
    lib = load()
    c = hp_config()
    lib.hp_config_default(C.byref(c))
    c.num_vw, c.Nm, c.D, c.waves = cfg.num_vw, cfg.Nm, cfg.D, cfg.waves
    c.nparams = cfg.nparams
    c.lr, c.momentum, c.seed = cfg.lr, cfg.momentum, cfg.seed
    c.grad_mode, c.w0_mode = cfg.grad_mode, cfg.w0_mode
    c.pull_policy, c.local_semantics = cfg.pull_policy, cfg.local_semantics
    c.conv_a, c.conv_sigma = getattr(cfg, "conv_a", 0.5), getattr(cfg, "conv_sigma", 1.0)
    c.update_freq = getattr(cfg, "F", 1)
    c.lr_schedule = getattr(cfg, "lr_schedule", 0)
    bounds = overrides.pop("ps_bounds", None)
    for k, v in overrides.items():
        setattr(c, k, v)
    if bounds is not None:
        arr = (C.c_int64 * len(bounds))(*[int(x) for x in bounds])
        c._ps_keep = arr                       # alive as long as the config
        c._ps_list = [int(x) for x in bounds]
        c.ps_bounds = C.cast(arr, C.c_void_p)
    if c.param_count < 0:
        c.param_count = c.nparams - c.param_begin
    return c


class Context:
    """One hp_ctx (one rank). Methods carry the C names without the prefix."""

    def __init__(self, cfg: hp_config, lib: Optional[C.CDLL] = None):
        self.lib = lib if lib is not None else load()
        self.cfg = cfg
        h = C.c_void_p()
        st = self.lib.hp_init_ex(C.byref(h), C.byref(cfg))
        if st != HP_OK:
            raise HetPipeError(st, self.lib.hp_last_error(None).decode())
        self.h = h

    # -- status handling ------------------------------------------------------
    def _chk(self, st: int, allow_block: bool = False) -> int:
        if st == HP_OK or (allow_block and st == HP_WOULD_BLOCK):
            return st
        raise HetPipeError(st, (self.lib.hp_last_error(self.h) or b"").decode())

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hp_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- protocol -------------------------------------------------------------
    def accumulate_minibatch(self, vw: int, p: int, grad_ptr: int = 0) -> int:
        return self._chk(self.lib.hp_accumulate_minibatch(self.h, vw, p, grad_ptr or None))

    def accumulate_minibatch_host(self, vw: int, p: int, host: np.ndarray) -> int:
        assert host.dtype == np.float32 and host.flags.c_contiguous
        return self._chk(self.lib.hp_accumulate_minibatch_host(
            self.h, vw, p, host.ctypes.data_as(C.c_void_p)))

    def push_wave(self, vw: int, c: int) -> int:
        return self._chk(self.lib.hp_push_wave(self.h, vw, c))

    def clock(self, vw: int):
        cl, cg = C.c_int64(), C.c_int64()
        st = self._chk(self.lib.hp_clock(self.h, vw, C.byref(cl), C.byref(cg)), True)
        return cl.value, cg.value, st == HP_WOULD_BLOCK

    def pull(self, vw: int) -> int:
        return self._chk(self.lib.hp_pull(self.h, vw), allow_block=True)

    def tick_end(self) -> int:
        return self._chk(self.lib.hp_tick_end(self.h))

    def flush(self) -> int:
        return self._chk(self.lib.hp_flush(self.h))

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        self._chk(self.lib.hp_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, handles: Sequence[bytes], comm_id: bytes) -> None:
        hb = C.create_string_buffer(b"".join(handles), 64 * len(handles))
        cb = C.create_string_buffer(comm_id, 128)
        self._chk(self.lib.hp_connect(self.h, hb, cb))

    def connect_symmetric(self, bases: Sequence[int], mc_base: int,
                          comm_id: Optional[bytes]) -> None:
        """comm_id None: co-located ranks without an NCCL communicator (K7 flag
        barriers, PEER exchange; include/hetpipe.h hp_connect_symmetric)."""
        arr = (C.c_void_p * len(bases))(*bases)
        cb = None if comm_id is None else C.create_string_buffer(comm_id, 128)
        self._chk(self.lib.hp_connect_symmetric(self.h, arr, mc_base or None, cb))

    def set_tick(self, t: int) -> int:
        return self._chk(self.lib.hp_set_tick(self.h, t))

    # -- controller -----------------------------------------------------------
    def schedule_begin(self, tau: Sequence[int], lat: Optional[Sequence[int]] = None) -> None:
        self._tau = np.ascontiguousarray(tau, dtype=np.int64)
        self._lat = None if lat is None else np.ascontiguousarray(lat, dtype=np.int64)
        self._chk(self.lib.hp_schedule_begin(
            self.h, self._tau.ctypes.data_as(C.c_void_p),
            None if self._lat is None else self._lat.ctypes.data_as(C.c_void_p)))

    def schedule_advance(self, target_commits: int) -> int:
        n = C.c_int64()
        self._chk(self.lib.hp_schedule_advance(self.h, target_commits, C.byref(n)))
        return n.value

    def run_schedule(self, tau: Sequence[int], lat: Optional[Sequence[int]] = None) -> None:
        t = np.ascontiguousarray(tau, dtype=np.int64)
        l_ = None if lat is None else np.ascontiguousarray(lat, dtype=np.int64)
        self._chk(self.lib.hp_run_schedule(
            self.h, t.ctypes.data_as(C.c_void_p),
            None if l_ is None else l_.ctypes.data_as(C.c_void_p)))

    def schedule_capture(self, target_commits: int) -> "Graph":
        """hp_schedule_capture: advance the controller now, capture the device
        work into a CUDA graph; Graph.launch() runs it (once)."""
        n, g = C.c_int64(), C.c_void_p()
        self._chk(self.lib.hp_schedule_capture(self.h, target_commits, C.byref(n), C.byref(g)))
        return Graph(self, g)

    def launch_floor(self, n: int = 1000, graph: bool = False) -> float:
        """hp_launch_floor: device us per empty launch (direct or in a graph)."""
        us = C.c_float()
        self._chk(self.lib.hp_launch_floor(self.h, n, 1 if graph else 0, C.byref(us)))
        return us.value

    def schedule_set_host_grads(self, bufs: Sequence[np.ndarray]) -> None:
        self._host_bufs = list(bufs)
        arr = (C.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
        self._host_ptrs = arr
        self._chk(self.lib.hp_schedule_set_host_grads(self.h, arr, len(bufs)))

    # -- data -----------------------------------------------------------------
    def local_len(self, which: int) -> int:
        """Length of buffer `which` on this rank (placement-aware)."""
        from workloads import even_shards
        c = self.cfg
        if c.world <= 1:
            return c.param_count
        if which < 0:
            from workloads import ceil_shards
            b = (getattr(c, "_ps_list", None)
                 or (ceil_shards if c.transport == XPORT_NCCL and c.vw_span == 1
                     else even_shards)(c.nparams, c.world))
            return b[c.rank + 1] - b[c.rank]
        for j in range(c.vw_span):
            if (which * c.vw_span + j) % c.world == c.rank:
                b = even_shards(c.nparams, c.vw_span)
                return b[j + 1] - b[j]
        return 0

    def sync(self) -> None:
        self._chk(self.lib.hp_sync(self.h))

    def drain(self) -> None:
        """hp_drain: launched work finished; deferred applies stay deferred."""
        self._chk(self.lib.hp_drain(self.h))

    def read_weights(self, which: int, offset: int = 0, count: Optional[int] = None,
                     out: Optional[np.ndarray] = None) -> np.ndarray:
        if count is None:
            count = self.local_len(which) - offset
        if out is None:
            out = np.empty(count, dtype=np.float32)
        self._chk(self.lib.hp_read_weights(self.h, which, offset, count,
                                           out.ctypes.data_as(C.c_void_p)))
        return out

    def trace_dump(self, path: str) -> None:
        self._chk(self.lib.hp_trace_dump(self.h, path.encode()))

    def trace_lines(self, tmp_path: str) -> list:
        self.trace_dump(tmp_path)
        with open(tmp_path) as f:
            return f.read().splitlines()

    def trace_enable(self, on: bool) -> None:
        self._chk(self.lib.hp_trace_enable(self.h, 1 if on else 0))

    def stats(self) -> hp_stats:
        s = hp_stats()
        self._chk(self.lib.hp_get_stats(self.h, C.byref(s)))
        return s

    def profile_enable(self, on: bool) -> None:
        self._chk(self.lib.hp_profile_enable(self.h, 1 if on else 0))

    def profile_read(self):
        ms, b, n = C.c_double(), C.c_double(), C.c_int64()
        self._chk(self.lib.hp_profile_read(self.h, C.byref(ms), C.byref(b), C.byref(n)))
        return ms.value, b.value, n.value


class Graph:
    """A captured controller advance (hp_graph); launch() once, then free."""

    def __init__(self, ctx: Context, g: C.c_void_p):
        self.ctx, self.g = ctx, g

    def launch(self) -> None:
        self.ctx._chk(self.ctx.lib.hp_graph_launch(self.g))

    def close(self) -> None:
        if self.g:
            self.ctx.lib.hp_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _profile_launches(self, max_records: int = 1 << 16):
    ms = np.zeros(max_records, dtype=np.float32)
    by = np.zeros(max_records, dtype=np.float64)
    sh = np.zeros(max_records, dtype=np.int32)
    sy = np.zeros(max_records, dtype=np.float64)
    t0 = np.zeros(max_records, dtype=np.float32)
    n = C.c_int64()
    self._chk(self.lib.hp_profile_launches(self.h, max_records, ms.ctypes.data_as(C.c_void_p),
                                           by.ctypes.data_as(C.c_void_p),
                                           sh.ctypes.data_as(C.c_void_p),
                                           sy.ctypes.data_as(C.c_void_p),
                                           t0.ctypes.data_as(C.c_void_p), C.byref(n)))
    k = n.value
    return ms[:k], by[:k], sh[:k], sy[:k], t0[:k]


Context.profile_launches = _profile_launches


def _profile_sync_latency(self, max_records: int = 1 << 16):
    ms = np.zeros(max_records, dtype=np.float32)
    vw = np.zeros(max_records, dtype=np.int32)
    waited = np.zeros(max_records, dtype=np.int32)
    n = C.c_int64()
    self._chk(self.lib.hp_profile_sync_latency(self.h, max_records, ms.ctypes.data_as(C.c_void_p),
                                               vw.ctypes.data_as(C.c_void_p),
                                               waited.ctypes.data_as(C.c_void_p), C.byref(n)))
    return ms[:n.value], vw[:n.value], waited[:n.value]


Context.profile_sync_latency = _profile_sync_latency


def _profile_link(self, max_records: int = 1 << 16):
    out = np.zeros(max_records, dtype=np.float64)
    n = C.c_int64()
    self._chk(self.lib.hp_profile_link(self.h, max_records, out.ctypes.data_as(C.c_void_p),
                                       C.byref(n)))
    return out[:n.value]


Context.profile_link = _profile_link


def _profile_streams(self, max_records: int = 1 << 16):
    out = np.zeros(max_records, dtype=np.int32)
    n = C.c_int64()
    self._chk(self.lib.hp_profile_streams(self.h, max_records, out.ctypes.data_as(C.c_void_p),
                                          C.byref(n)))
    return out[:n.value]


Context.profile_streams = _profile_streams


def comm_unique_id(lib: Optional[C.CDLL] = None) -> bytes:
    lib = lib if lib is not None else load()
    buf = C.create_string_buffer(128)
    st = lib.hp_comm_unique_id(buf)
    if st != HP_OK:
        raise HetPipeError(st, lib.hp_last_error(None).decode())
    return buf.raw


def arena_bytes(cfg: hp_config, lib: Optional[C.CDLL] = None) -> int:
    n = (lib if lib is not None else load()).hp_arena_bytes(C.byref(cfg))
    if n < 0:
        raise HetPipeError(HP_ERR_INVALID, "hp_arena_bytes: bad config")
    return n


def s_global(Nm: int, D: int) -> int:
    return load().hp_s_global(Nm, D)


def version_floor(p: int, Nm: int, D: int) -> int:
    return load().hp_version_floor(p, Nm, D)


# ---- intra-VW pipeline schedule (include/hetpipe.h hp_partition & co.) -------
def _units(units):
    arr = (hp_unit * len(units))()
    for i, u in enumerate(units):
        arr[i] = hp_unit(u.params, u.fwd_flops, u.act_out, u.act_resident)
    return arr


def _gpus(gpus):
    arr = (hp_gpu * len(gpus))()
    for i, g in enumerate(gpus):
        arr[i] = hp_gpu(g["flops"], g["mem"], g["node"], 0)
    return arr


def partition(units, gpus, Nm: int, batch: int = 32, intra_bps: float = 15.75e9,
              inter_bps: float = 56e9 / 8, lib: Optional[C.CDLL] = None):
    """(bottleneck_ns, order, cuts, stage_costs) or None if nothing fits.
    units: objects with params/fwd_flops/act_out/act_resident; gpus: dicts
    {"flops", "mem", "node"}."""
    lib = lib if lib is not None else load()
    k = len(gpus)
    order = (C.c_int32 * k)()
    cuts = (C.c_int32 * (k + 1))()
    costs = (C.c_int64 * (4 * k))()
    b = C.c_int64()
    st = lib.hp_partition(_units(units), len(units), _gpus(gpus), k, Nm, batch, intra_bps,
                          inter_bps, order, cuts, costs, C.byref(b))
    if st == HP_WOULD_BLOCK:
        return None
    if st != HP_OK:
        raise HetPipeError(st, "hp_partition: bad arguments")
    return (b.value, tuple(order), tuple(cuts),
            [tuple(costs[4 * q:4 * q + 4]) for q in range(k)])


def max_m(units, gpus, batch: int = 32, intra_bps: float = 15.75e9,
          inter_bps: float = 56e9 / 8, lib: Optional[C.CDLL] = None) -> int:
    lib = lib if lib is not None else load()
    return lib.hp_max_m(_units(units), len(units), _gpus(gpus), len(gpus), batch, intra_bps,
                        inter_bps)


def _costs(costs):
    flat = [int(x) for c in costs for x in c]
    return (C.c_int64 * len(flat))(*flat)


def pipeline_simulate(costs, Nm: int, P: int, lib: Optional[C.CDLL] = None):
    """(start_ns[P], complete_ns[P]) of minibatches 1..P."""
    lib = lib if lib is not None else load()
    s = np.zeros(P, dtype=np.int64)
    c = np.zeros(P, dtype=np.int64)
    st = lib.hp_pipeline_simulate(_costs(costs), len(costs), Nm, P, s.ctypes.data_as(C.c_void_p),
                                  c.ctypes.data_as(C.c_void_p))
    if st != HP_OK:
        raise HetPipeError(st, "hp_pipeline_simulate: bad arguments")
    return s, c


def pipeline_tau_latency(costs, Nm: int, P: int = 0, lib: Optional[C.CDLL] = None):
    lib = lib if lib is not None else load()
    t, l_ = C.c_int64(), C.c_int64()
    st = lib.hp_pipeline_tau_latency(_costs(costs), len(costs), Nm, P, C.byref(t), C.byref(l_))
    if st != HP_OK:
        raise HetPipeError(st, "hp_pipeline_tau_latency: bad arguments")
    return t.value, l_.value
