"""Thin ctypes binding of libnacs (include/nacs.h): argument marshalling only.

Every step of the ranking and placement runs in the CUDA kernels of libnacs.so; this
module converts numpy arrays / torch tensors to pointers and back.  There is no
fallback: if libnacs.so is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NACS_LIB", os.path.join(HERE, "libnacs.so"))  # NACS_LIB: experiment builds

NACS_OK, NACS_EINVAL, NACS_ENOMEM, NACS_ECUDA, NACS_ENCCL, NACS_ENOTOPO, NACS_ETOOBIG = range(7)
STATUS_NAMES = ["OK", "EINVAL", "ENOMEM", "ECUDA", "ENCCL", "ENOTOPO", "ETOOBIG"]
NACS_AHP, NACS_TOPSIS, NACS_BF, NACS_WF = 0, 1, 2, 3
NACS_DEVICE_PTRS, NACS_ASYNC, NACS_EXACT_FP64 = 1, 2, 4
NACS_RANK_PER_POD, NACS_RANK_ONCE = 0, 1
MAX_CONTAINERS, MAX_VLINKS, MAX_K = 128, 512, 64

# Table 4: weights over (CPU, RAM, Fragmentation, Bandwidth)
SCHEMAS = {"flat": (0.25, 0.25, 0.25, 0.25),
           "clustering": (0.17, 0.17, 0.5, 0.16),
           "network": (0.17, 0.17, 0.16, 0.5)}
METHODS = {"ahp": NACS_AHP, "topsis": NACS_TOPSIS, "bf": NACS_BF, "wf": NACS_WF}

P32 = C.POINTER(C.c_int32)
PU8 = C.POINTER(C.c_uint8)
PF = C.POINTER(C.c_float)


class Topology(C.Structure):
    _fields_ = [("k", C.c_int32), ("cpu_cap", C.c_int32), ("ram_cap", C.c_int32), ("link_cap", C.c_int32),
                ("cpu_res", C.c_void_p), ("ram_res", C.c_void_p), ("active", C.c_void_p),
                ("link_res", C.c_void_p)]


class PodQuery(C.Structure):
    _fields_ = [("cpu_demand", C.c_int32), ("ram_demand", C.c_int32), ("n_flows", C.c_int32),
                ("flow_server", C.c_void_p), ("flow_bw", C.c_void_p), ("n_excluded", C.c_int32),
                ("excluded", C.c_void_p)]


class Requests(C.Structure):
    _fields_ = [("n_requests", C.c_int32), ("container_off", C.c_void_p), ("cpu_min", C.c_void_p),
                ("cpu_max", C.c_void_p), ("ram_min", C.c_void_p), ("ram_max", C.c_void_p),
                ("pod_of", C.c_void_p), ("vlink_off", C.c_void_p), ("vl_src", C.c_void_p),
                ("vl_dst", C.c_void_p), ("bw_min", C.c_void_p), ("bw_max", C.c_void_p)]


class Placements(C.Structure):
    _fields_ = [("status", C.c_void_p), ("server_of_container", C.c_void_p), ("cpu_alloc", C.c_void_p),
                ("ram_alloc", C.c_void_p), ("bw_alloc", C.c_void_p), ("path_of_vlink", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("method", C.c_int), ("weights", C.c_double * 4), ("ahp_rule", C.c_int32),
                ("l1_mode", C.c_int32), ("path_filter", C.c_int32), ("flags", C.c_uint32),
                ("rank_mode", C.c_int32), ("bw_criterion", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("pod_steps", C.c_int64), ("servers_ranked", C.c_int64), ("retries", C.c_int64),
                ("fp64_decisions", C.c_int64), ("invalid", C.c_int64), ("feasible", C.c_int64),
                ("ahp_pairs", C.c_int64), ("scanned_a", C.c_int64), ("scanned_b", C.c_int64),
                ("edges_scanned", C.c_int64), ("bfs_runs", C.c_int64)]


class SimConfig(C.Structure):
    _fields_ = [("max_ticks", C.c_int32), ("hol_blocking", C.c_int32)]


class SimReport(C.Structure):
    _fields_ = [("start_tick", C.c_void_p), ("attempts", C.c_void_p), ("tick_servers", C.c_void_p),
                ("tick_links", C.c_void_p), ("tick_queue", C.c_void_p), ("events", C.c_int64),
                ("attempts_total", C.c_int64), ("accepted", C.c_int64), ("sched_seconds", C.c_double),
                ("wall_seconds", C.c_double)]


class Graph(C.Structure):
    _fields_ = [("n_vertices", C.c_int32), ("n_servers", C.c_int32), ("n_links", C.c_int32),
                ("link_u", C.c_void_p), ("link_v", C.c_void_p), ("link_res", C.c_void_p)]


class PathQuery(C.Structure):
    _fields_ = [("n_queries", C.c_int32), ("src", C.c_void_p), ("dst", C.c_void_p), ("demand", C.c_void_p)]


EXPORTS = ["nacs_create", "nacs_create_sharded", "nacs_nccl_unique_id", "nacs_destroy", "nacs_load_topology",
           "nacs_read_topology", "nacs_rank_ahp", "nacs_rank_topsis", "nacs_rank_topsis_many", "nacs_schedule_request",
           "nacs_schedule_batch", "nacs_last_stats", "nacs_last_error", "nacs_load_graph", "nacs_widest_paths",
           "nacs_logical_bandwidth", "nacs_release", "nacs_simulate"]

_lib = None


def lib():
    """Load libnacs.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1909_07673_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.nacs_create.argtypes = [C.POINTER(vp), C.c_int, vp]
        L.nacs_create_sharded.argtypes = [C.POINTER(vp), C.c_int, vp, vp, C.c_int, C.c_int]
        L.nacs_nccl_unique_id.argtypes = [vp]
        L.nacs_destroy.argtypes = [vp]
        L.nacs_destroy.restype = None
        L.nacs_load_topology.argtypes = [vp, C.POINTER(Topology)]
        L.nacs_read_topology.argtypes = [vp, vp, vp, vp, vp]
        for f in (L.nacs_rank_ahp, L.nacs_rank_topsis):
            f.argtypes = [vp, C.POINTER(Options), C.POINTER(PodQuery), vp, vp, vp]
        L.nacs_rank_topsis_many.argtypes = [vp, C.POINTER(Options), C.POINTER(PodQuery), C.c_int32, vp, C.c_int64,
                                            vp, vp, vp]
        for f in (L.nacs_schedule_request, L.nacs_schedule_batch):
            f.argtypes = [vp, C.POINTER(Options), C.POINTER(Requests), C.POINTER(Placements)]
        L.nacs_last_stats.argtypes = [vp, C.POINTER(Stats)]
        L.nacs_release.argtypes = [vp, C.c_uint32, C.POINTER(Requests), C.POINTER(Placements)]
        L.nacs_simulate.argtypes = [vp, C.POINTER(Options), C.POINTER(Requests), vp, vp, C.POINTER(SimConfig),
                                    C.POINTER(Placements), C.POINTER(SimReport)]
        L.nacs_load_graph.argtypes = [vp, C.POINTER(Graph)]
        L.nacs_widest_paths.argtypes = [vp, C.POINTER(PathQuery), C.c_uint32, vp, vp, vp, C.c_int32]
        L.nacs_logical_bandwidth.argtypes = [vp, C.c_uint32, vp]
        L.nacs_last_error.argtypes = [vp]
        L.nacs_last_error.restype = C.c_char_p
        for name in EXPORTS:
            if name not in ("nacs_destroy", "nacs_last_error"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


class NacsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


def _np_ptr(a):
    return None if a is None else a.ctypes.data


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return a.data_ptr()
    return a.ctypes.data


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


REQ_KEYS = ("container_off", "cpu_min", "cpu_max", "ram_min", "ram_max", "pod_of", "vlink_off", "vl_src",
            "vl_dst", "bw_min", "bw_max")
OUT_KEYS = ("status", "server_of_container", "cpu_alloc", "ram_alloc", "bw_alloc", "path_of_vlink")


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 makes it; the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    st = lib().nacs_nccl_unique_id(buf)
    if st != NACS_OK:
        raise NacsError(st, "ncclGetUniqueId failed")
    return buf.raw


class Context:
    """One libnacs context on one CUDA device (one per process / rank).

    shard=(rank, world, uid): server-sharded sequential scheduling over `world` ranks
    (uid = nccl_unique_id() from rank 0, or None for loopback shards on this device)."""

    def __init__(self, device: int = 0, stream=None, shard=None):
        self._lib = lib()
        self._h = C.c_void_p()
        handle = None
        if stream is not None:
            handle = stream if isinstance(stream, int) else stream.cuda_stream
        if shard is None:
            st = self._lib.nacs_create(C.byref(self._h), device, handle)
        else:
            rank, world, uid = shard
            ub = None if uid is None else C.create_string_buffer(bytes(uid), 128)
            st = self._lib.nacs_create_sharded(C.byref(self._h), device, handle, ub, int(rank), int(world))
        if st != NACS_OK:
            raise NacsError(st, "nacs_create failed (no CUDA device?)")
        self.device = device
        self.k = None

    def close(self):
        if self._h:
            self._lib.nacs_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != NACS_OK:
            raise NacsError(st, self._lib.nacs_last_error(self._h).decode())

    # ------------------------------------------------------------- topology --
    def load_topology(self, snap: dict):
        k = int(snap["k"])
        keep = [None if snap.get(key) is None else np.ascontiguousarray(snap[key], dtype=dt)
                for key, dt in (("cpu_res", np.int32), ("ram_res", np.int32), ("active", np.uint8),
                                ("link_res", np.int32))]
        t = Topology(k, int(snap["cpu_cap"]), int(snap["ram_cap"]), int(snap["link_cap"]),
                     *[_np_ptr(a) for a in keep])
        self._check(self._lib.nacs_load_topology(self._h, C.byref(t)))
        self.k = k
        self.n = k ** 3 // 4
        self.L = 3 * self.n

    def read_topology(self) -> dict:
        cpu = np.zeros(self.n, np.int32)
        ram = np.zeros(self.n, np.int32)
        act = np.zeros(self.n, np.uint8)
        link = np.zeros(self.L, np.int32)
        self._check(self._lib.nacs_read_topology(self._h, _np_ptr(cpu), _np_ptr(ram), _np_ptr(act),
                                                 _np_ptr(link)))
        return dict(cpu_res=cpu, ram_res=ram, active=act, link_res=link)

    # -------------------------------------------------------------- options --
    @staticmethod
    def options(method, weights, ahp_rule=0, l1_mode=0, path_filter=1, flags=0, rank_once=False,
                bw_criterion=0) -> Options:
        if isinstance(weights, str):
            weights = SCHEMAS[weights]
        m = METHODS[method] if isinstance(method, str) else int(method)
        return Options(m, (C.c_double * 4)(*[float(w) for w in weights]), ahp_rule, l1_mode, path_filter, flags,
                       NACS_RANK_ONCE if rank_once else NACS_RANK_PER_POD, int(bw_criterion))

    # ---------------------------------------------------------------- rank ---
    def rank(self, method, weights, dem_cpu, dem_ram, flows=(), excluded=(), exact64=False, **kw) -> dict:
        """One pod step on the current state: returns mask (uint8[n]), scores (float32[n]), best."""
        o = self.options(method, weights, flags=NACS_EXACT_FP64 if exact64 else 0, **kw)
        fv = _i32([f[0] for f in flows]) if len(flows) else np.zeros(1, np.int32)
        fd = _i32([f[1] for f in flows]) if len(flows) else np.zeros(1, np.int32)
        ex = _i32(list(excluded)) if len(excluded) else np.zeros(1, np.int32)
        q = PodQuery(int(dem_cpu), int(dem_ram), len(flows), _np_ptr(fv), _np_ptr(fd), len(excluded), _np_ptr(ex))
        mask = np.zeros(self.n, np.uint8)
        scores = np.zeros(self.n, np.float32)
        best = np.zeros(1, np.int32)
        fn = self._lib.nacs_rank_ahp if o.method == NACS_AHP else self._lib.nacs_rank_topsis
        self._check(fn(self._h, C.byref(o), C.byref(q), _np_ptr(mask), _np_ptr(scores), _np_ptr(best)))
        return dict(mask=mask, scores=scores, best=int(best[0]))

    def rank_many(self, states, dem_cpu, dem_ram, flows=(), excluded=(), weights="flat", scores=True, mask=True,
                  out=None, flags=0, exact64=False, **kw) -> dict:
        """TOPSIS ranking of one pod step on each of B DC states (nacs_rank_topsis_many).

        states: int32 [B, words] (words >= 3n + L: cpu | ram | active | links per row), a numpy
        array (host path) or a contiguous torch CUDA tensor (device path, one launch).
        out: optional preallocated dict(mask [B, n] uint8, scores [B, n] float32, best [B] int32)
        of the same kind.  Returns that dict."""
        dev = _is_torch(states)
        if states.ndim != 2 or states.shape[1] < 3 * self.n + self.L:
            raise ValueError(f"states: shape [B, >= {3 * self.n + self.L}] expected")
        B = int(states.shape[0])
        if dev:
            import torch
            self._check_tensor("states", states)
            if states.stride(1) != 1:
                raise ValueError("states: rows must be contiguous")
            stride = int(states.stride(0))
            flags |= NACS_DEVICE_PTRS
            if out is None:
                d = states.device
                out = dict(mask=torch.empty((B, self.n), dtype=torch.uint8, device=d) if mask else None,
                           scores=torch.empty((B, self.n), dtype=torch.float32, device=d) if scores else None,
                           best=torch.empty(B, dtype=torch.int32, device=d))
            mk = lambda xs: torch.tensor(list(xs), dtype=torch.int32, device=states.device) if len(xs) else None
            fv, fd, ex = mk([f[0] for f in flows]), mk([f[1] for f in flows]), mk(excluded)
        else:
            states = np.ascontiguousarray(states, dtype=np.int32)
            stride = states.shape[1]
            if out is None:
                out = dict(mask=np.zeros((B, self.n), np.uint8) if mask else None,
                           scores=np.zeros((B, self.n), np.float32) if scores else None,
                           best=np.zeros(B, np.int32))
            fv = _i32([f[0] for f in flows]) if len(flows) else np.zeros(1, np.int32)
            fd = _i32([f[1] for f in flows]) if len(flows) else np.zeros(1, np.int32)
            ex = _i32(list(excluded)) if len(excluded) else np.zeros(1, np.int32)
        o = self.options("topsis", weights, flags=flags | (NACS_EXACT_FP64 if exact64 else 0), **kw)
        q = PodQuery(int(dem_cpu), int(dem_ram), len(flows), _ptr(fv), _ptr(fd), len(excluded), _ptr(ex))
        self._check(self._lib.nacs_rank_topsis_many(self._h, C.byref(o), C.byref(q), B, _ptr(states), stride,
                                                    _ptr(out["mask"]), _ptr(out["scores"]), _ptr(out["best"])))
        return out

    # ------------------------------------------------------------ schedule ---
    def _check_tensor(self, key, a, min_numel=None, exact_numel=None):
        """A torch tensor handed to the library by pointer must be int32, contiguous and on
        this context's device, and hold at least the elements the kernels will touch."""
        import torch
        if a.dtype != torch.int32:
            raise ValueError(f"{key}: dtype {a.dtype}, expected torch.int32")
        if not a.is_contiguous():
            raise ValueError(f"{key}: not contiguous")
        if a.device.type != "cuda" or a.device.index != self.device:
            raise ValueError(f"{key}: on {a.device}, expected cuda:{self.device}")
        if exact_numel is not None and a.numel() != exact_numel:
            raise ValueError(f"{key}: {a.numel()} elements, expected {exact_numel}")
        if min_numel is not None and a.numel() < min_numel:
            raise ValueError(f"{key}: {a.numel()} elements, at least {min_numel} needed")

    def _requests(self, reqs: dict):
        arrs = []
        dev = None
        for key in REQ_KEYS:
            a = reqs[key]
            if _is_torch(a):
                dev = True if dev in (None, True) else "mixed"
                arrs.append(a)
            else:
                dev = False if dev in (None, False) else "mixed"
                arrs.append(_i32(a))
        if dev == "mixed":
            raise ValueError("request arrays must be all host or all device")
        R = int(reqs["n_requests"])
        if R < 0:
            raise ValueError("n_requests < 0")
        by_key = dict(zip(REQ_KEYS, arrs))
        if dev:
            import torch
            for key, a in by_key.items():  # dtype and layout of every array before devices and sizes
                if a.dtype != torch.int32:
                    raise ValueError(f"{key}: dtype {a.dtype}, expected torch.int32")
                if not a.is_contiguous():
                    raise ValueError(f"{key}: not contiguous")
            # container_off[R] / vlink_off[R] live on the device: the per-container and per-vlink
            # arrays must agree in length with each other (their common length bounds the offsets)
            for key in ("container_off", "vlink_off"):
                self._check_tensor(key, by_key[key], exact_numel=R + 1)
            for group in (("cpu_min", "cpu_max", "ram_min", "ram_max", "pod_of"), ("vl_src", "vl_dst", "bw_min", "bw_max")):
                for key in group:
                    self._check_tensor(key, by_key[key], exact_numel=by_key[group[0]].numel())
            sizes = dict(R=R, C=by_key["cpu_min"].numel(), V=by_key["vl_src"].numel())
        else:
            for key in ("container_off", "vlink_off"):
                if by_key[key].size != R + 1:
                    raise ValueError(f"{key}: {by_key[key].size} elements, expected n_requests + 1 = {R + 1}")
            Cn, Vn = int(by_key["container_off"][-1]), int(by_key["vlink_off"][-1])
            for key, need in (("cpu_min", Cn), ("cpu_max", Cn), ("ram_min", Cn), ("ram_max", Cn), ("pod_of", Cn),
                              ("vl_src", Vn), ("vl_dst", Vn), ("bw_min", Vn), ("bw_max", Vn)):
                if by_key[key].size < need:
                    raise ValueError(f"{key}: {by_key[key].size} elements, at least {need} needed")
            sizes = dict(R=R, C=Cn, V=Vn)
        self._req_sizes = sizes
        r = Requests(R, *[_ptr(a) for a in arrs])
        return r, arrs, bool(dev)

    def _check_out(self, out: dict, device: bool):
        """Caller-supplied output arrays: int32, contiguous, on the right side, large enough."""
        s = self._req_sizes
        need = dict(status=s["R"], server_of_container=s["C"], cpu_alloc=s["C"], ram_alloc=s["C"], bw_alloc=s["V"],
                    path_of_vlink=s["V"])
        for key in OUT_KEYS:
            a = out[key]
            if device:
                if not _is_torch(a):
                    raise ValueError(f"out[{key}]: device requests need torch CUDA outputs")
                self._check_tensor(f"out[{key}]", a, min_numel=need[key])
            else:
                if _is_torch(a) or not isinstance(a, np.ndarray):
                    raise ValueError(f"out[{key}]: host requests need numpy outputs")
                if a.dtype != np.int32 or not a.flags.c_contiguous or not a.flags.writeable:
                    raise ValueError(f"out[{key}]: must be a writeable C-contiguous int32 array")
                if a.size < need[key]:
                    raise ValueError(f"out[{key}]: {a.size} elements, at least {need[key]} needed")

    def _alloc_out(self, reqs: dict, device: bool):
        R = int(reqs["n_requests"])
        Cn = int(reqs["container_off"][-1]) if len(reqs["container_off"]) else 0
        Vn = int(reqs["vlink_off"][-1]) if len(reqs["vlink_off"]) else 0
        sizes = dict(status=R, server_of_container=Cn, cpu_alloc=Cn, ram_alloc=Cn, bw_alloc=Vn, path_of_vlink=Vn)
        if device:
            import torch
            out = {k: torch.empty(max(v, 1), dtype=torch.int32, device=f"cuda:{self.device}") for k, v in sizes.items()}
        else:
            out = {k: np.zeros(max(v, 1), np.int32) for k, v in sizes.items()}
        return out, sizes

    def _schedule(self, fn, reqs, method, weights, out=None, flags=0, **kw) -> dict:
        r, keep, dev = self._requests(reqs)
        if dev:
            flags |= NACS_DEVICE_PTRS
        o = self.options(method, weights, flags=flags, **kw)
        sizes = None
        if out is None:
            out, sizes = self._alloc_out(reqs, dev)
        else:
            self._check_out(out, dev)
        p = Placements(*[_ptr(out[k]) for k in OUT_KEYS])
        self._check(fn(self._h, C.byref(o), C.byref(r), C.byref(p)))
        del keep
        if sizes is not None:
            out = {k: out[k][: sizes[k]] for k in OUT_KEYS}
        return out

    def schedule_request(self, reqs: dict, method, weights, out=None, flags=0, **kw) -> dict:
        """Requests in order against the live state; accepted requests stay committed."""
        return self._schedule(self._lib.nacs_schedule_request, reqs, method, weights, out, flags, **kw)

    def schedule_batch(self, reqs: dict, method, weights, out=None, flags=0, **kw) -> dict:
        """Every request against the same snapshot (snapshot isolation); the state is unchanged."""
        return self._schedule(self._lib.nacs_schedule_batch, reqs, method, weights, out, flags, **kw)

    # ------------------------------------------------- departures, simulator ---
    def release(self, reqs: dict, placements: dict, flags=0):
        """Departure of every accepted request (status 1) of `reqs` (placements as returned)."""
        r, keep, dev = self._requests(reqs)
        if dev:
            flags |= NACS_DEVICE_PTRS
            self._check_out(placements, True)
            outs = [placements[k] for k in OUT_KEYS]
        else:
            outs = [_i32(placements[k]) for k in OUT_KEYS]
            self._check_out(dict(zip(OUT_KEYS, outs)), False)
        p = Placements(*[_ptr(a) for a in outs])
        self._check(self._lib.nacs_release(self._h, flags, C.byref(r), C.byref(p)))
        del keep

    def simulate(self, reqs: dict, arrival, duration, method, weights, max_ticks: int, hol: int = 1, **kw) -> dict:
        """Discrete-event simulation on the live state (reading R28): per-request start / attempts,
        final placements, per-tick |N^s'|, |E^s'|, queue length, and totals."""
        r, keep, dev = self._requests(reqs)
        if dev:
            raise ValueError("simulate takes host arrays")
        o = self.options(method, weights, **kw)
        R = int(reqs["n_requests"])
        out, sizes = self._alloc_out(reqs, False)
        p = Placements(*[_ptr(out[k]) for k in OUT_KEYS])
        arr, dur = _i32(arrival), _i32(duration)
        start, att = np.zeros(max(R, 1), np.int32), np.zeros(max(R, 1), np.int32)
        ts, tl, tq = (np.zeros(max_ticks, np.int32) for _ in range(3))
        rep = SimReport(_np_ptr(start), _np_ptr(att), _np_ptr(ts), _np_ptr(tl), _np_ptr(tq), 0, 0, 0, 0.0, 0.0)
        cfg = SimConfig(int(max_ticks), int(hol))
        self._check(self._lib.nacs_simulate(self._h, C.byref(o), C.byref(r), _np_ptr(arr), _np_ptr(dur),
                                            C.byref(cfg), C.byref(p), C.byref(rep)))
        del keep
        T = int(rep.events)
        return dict(start=start[:R], attempts=att[:R], status=out["status"][:R],
                    placements={k: out[k][: sizes[k]] for k in OUT_KEYS},
                    tick_servers=ts[:T], tick_links=tl[:T], tick_queue=tq[:T],
                    totals=dict(events=T, attempts=int(rep.attempts_total), accepted=int(rep.accepted)),
                    sched_seconds=rep.sched_seconds, wall_seconds=rep.wall_seconds)

    # ----------------------------------------------------- general topology ---
    def load_graph(self, graph: dict):
        """An arbitrary undirected DC graph: dict(n_vertices, n_servers, link_u, link_v, link_res)."""
        keep = [_i32(graph[k]) for k in ("link_u", "link_v", "link_res")]
        g = Graph(int(graph["n_vertices"]), int(graph["n_servers"]), keep[0].size, *[_np_ptr(a) for a in keep])
        self._check(self._lib.nacs_load_graph(self._h, C.byref(g)))
        self.graph_V = int(graph["n_vertices"])
        self.graph_ns = int(graph["n_servers"])

    def widest_paths(self, src, dst, demand, max_hops=None, with_path=True, out=None, flags=0):
        """Widest-shortest path per (src, dst, demand) query (modified Dijkstra).
        numpy inputs -> numpy outputs (bottleneck, hops, path[nq, max_hops+1] or None); torch CUDA
        inputs -> torch outputs (device pointers).  out: preallocated (bn, hops, path) to reuse."""
        dev = _is_torch(src)
        if not dev:
            src, dst, demand = _i32(src), _i32(dst), _i32(demand)
        nq = int(src.numel() if dev else src.size)
        if dev:
            for key, a in (("src", src), ("dst", dst), ("demand", demand)):
                self._check_tensor(key, a, exact_numel=nq)
        elif dst.size != nq or demand.size != nq:
            raise ValueError("src, dst and demand must have the same length")
        if max_hops is None:
            max_hops = 16
        if out is None:
            if dev:
                import torch
                mk = lambda *shape: torch.empty(shape, dtype=torch.int32, device=src.device)
            else:
                mk = lambda *shape: np.zeros(shape, np.int32)
            out = (mk(max(nq, 1)), mk(max(nq, 1)), mk(max(nq, 1), max_hops + 1) if with_path else None)
        bn, hops, path = out
        for key, a, need in (("bottleneck", bn, nq), ("hops", hops, nq),
                             ("path", path, nq * (max_hops + 1))):
            if a is None:
                continue
            if dev:
                self._check_tensor(key, a, min_numel=need)
            elif (not isinstance(a, np.ndarray) or a.dtype != np.int32 or not a.flags.c_contiguous
                  or a.size < need):
                raise ValueError(f"{key}: must be a C-contiguous int32 array of at least {need} elements")
        q = PathQuery(nq, _ptr(src), _ptr(dst), _ptr(demand))
        if dev:
            flags |= NACS_DEVICE_PTRS
        self._check(self._lib.nacs_widest_paths(self._h, C.byref(q), flags, _ptr(bn), _ptr(hops), _ptr(path),
                                                int(max_hops)))
        return bn[:nq], hops[:nq], (None if path is None else path[:nq])

    def logical_bandwidth(self, out=None, flags=0):
        """R2 alternative criterion: int64[n_servers], sum of widest-shortest bottlenecks."""
        if out is None:
            out = np.zeros(self.graph_ns, np.int64)
        if _is_torch(out):
            import torch
            if out.dtype != torch.int64 or not out.is_contiguous() or out.numel() < self.graph_ns or \
                    out.device != torch.device("cuda", self.device):
                raise ValueError(f"out: a contiguous int64 cuda:{self.device} tensor of >= {self.graph_ns} elements")
            flags |= NACS_DEVICE_PTRS
        elif out.dtype != np.int64 or not out.flags.c_contiguous or out.size < self.graph_ns:
            raise ValueError(f"out: a C-contiguous int64 array of >= {self.graph_ns} elements")
        self._check(self._lib.nacs_logical_bandwidth(self._h, flags, _ptr(out)))
        return out

    def last_stats(self) -> dict:
        s = Stats()
        self._check(self._lib.nacs_last_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}
