"""B200-native Blink (arXiv:1910.04940): tree-packed Broadcast / AllReduce.

Thin Python binding over the C ABI in ``include/blink.h`` (``libblink.so``,
built in-tree by ``paper_1910_04940_b200.build``).  This module only marshals
arguments: every step of a collective runs in the library's sm_100a kernels.
There is no Python or CPU fallback -- importing fails loudly if the library is
missing.

Buffers may be given as torch tensors (their ``data_ptr()`` is passed) or as
raw device addresses (ints).  Streams are ``torch.cuda.Stream`` objects, raw
``cudaStream_t`` ints, or None (the current torch stream if torch is loaded,
else the legacy default stream).
"""
import ctypes
import json
import os

__all__ = ["BlinkError", "Comm", "Graph", "config", "plan_json", "init_all", "init_multiprocess",
           "DTYPES", "OPS", "LIB_PATH"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libblink.so")
from . import build as _build  # noqa: E402  (no package imports inside)
if _build._stale() and os.path.exists(_build.NVCC):
    _build.build()             # sources changed since the last build (dev checkout)
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1910_04940_b200.build` "
                      "(there is no fallback implementation)")
_lib = ctypes.CDLL(LIB_PATH)

DTYPES = {"f32": 0, "bf16": 1, "i32": 2}
ESIZE = {"f32": 4, "bf16": 2, "i32": 4}
OPS = {"sum": 0, "prod": 1, "min": 2, "max": 3, "avg": 4}
NODE_GPU, NODE_SWITCH = 0, 1


class _Link(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int), ("dst", ctypes.c_int), ("capacity", ctypes.c_double),
                ("bidirectional", ctypes.c_int)]


class _Graph(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int), ("kinds", ctypes.POINTER(ctypes.c_int)),
                ("num_links", ctypes.c_int), ("links", ctypes.POINTER(_Link))]


class _Config(ctypes.Structure):
    _fields_ = [("mwu_eps", ctypes.c_double), ("ilp_gap", ctypes.c_double),
                ("chunk_bytes", ctypes.c_size_t), ("ctas", ctypes.c_int), ("threads", ctypes.c_int),
                ("timeout_s", ctypes.c_double), ("onehop_bcast_max_bytes", ctypes.c_size_t),
                ("staging_bytes", ctypes.c_size_t), ("autotune", ctypes.c_int),
                ("launch_per_rank", ctypes.c_int), ("ll_max_bytes", ctypes.c_size_t),
                ("shallow_max_bytes", ctypes.c_size_t), ("nvls", ctypes.c_int),
                ("nvls_bytes", ctypes.c_size_t)]


class Miad(ctypes.Structure):
    """blink_miad_t: the MIAD chunk-size controller state."""
    _fields_ = [("chunk", ctypes.c_size_t), ("best", ctypes.c_size_t), ("init", ctypes.c_size_t),
                ("step", ctypes.c_size_t), ("min_chunk", ctypes.c_size_t),
                ("max_chunk", ctypes.c_size_t), ("last_thr", ctypes.c_double),
                ("best_thr", ctypes.c_double), ("tol", ctypes.c_double), ("phase", ctypes.c_int),
                ("iters", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("last_ctas", ctypes.c_int),
                ("last_chunks", ctypes.c_int), ("last_trees", ctypes.c_int),
                ("last_chunk_bytes", ctypes.c_int64), ("last_steal_channels", ctypes.c_int)]


_vp, _sz, _i, _cp = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_char_p
_SIGS = {
    "blink_config_default": (None, [ctypes.POINTER(_Config)]),
    "blink_plan_json": (_i, [ctypes.POINTER(_Graph), _i, ctypes.POINTER(_Config), _i, _i, _sz, _i,
                             _cp, ctypes.POINTER(_sz)]),
    "blink_init_all": (_i, [ctypes.POINTER(_vp), _i, ctypes.POINTER(_i), ctypes.POINTER(_Graph),
                            ctypes.POINTER(_Config)]),
    "blink_init": (_i, [ctypes.POINTER(_vp), _i, _i, _i, ctypes.POINTER(_Graph), ctypes.POINTER(_Config)]),
    "blink_export_handle": (_i, [_vp, _vp, ctypes.POINTER(_sz)]),
    "blink_connect": (_i, [_vp, _vp, _sz]),
    "blink_register_export": (_i, [_vp, _vp, _sz, _vp, ctypes.POINTER(_sz)]),
    "blink_register_connect": (_i, [_vp, _vp, _vp, _sz]),
    "blink_broadcast": (_i, [_vp, _vp, _vp, _sz, _i, _i, _vp]),
    "blink_allreduce": (_i, [_vp, _vp, _vp, _sz, _i, _i, _vp]),
    "blink_reduce_scatter": (_i, [_vp, _vp, _vp, _sz, _i, _i, _vp]),
    "blink_allgather": (_i, [_vp, _vp, _vp, _sz, _i, _vp]),
    "blink_gather": (_i, [_vp, _vp, _vp, _sz, _i, _i, _vp]),
    "blink_get_plan": (_i, [_vp, _i, _i, _sz, _i, _cp, ctypes.POINTER(_sz)]),
    "blink_get_stats": (_i, [_vp, ctypes.POINTER(_Stats)]),
    "blink_get_trace": (_i, [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(_sz)]),
    "blink_comm_info": (_i, [_vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "blink_destroy": (_i, [_vp]),
    "blink_miad_init": (None, [ctypes.POINTER(Miad), _sz, _sz, _sz]),
    "blink_miad_step": (_sz, [ctypes.POINTER(Miad), ctypes.c_double]),
    "blink_topology_json": (_i, [_i, ctypes.POINTER(_cp), _cp, ctypes.POINTER(_sz)]),
    "blink_hybrid_split": (_i, [_sz, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.POINTER(_sz), ctypes.POINTER(_sz)]),
    "blink_result_string": (_cp, [_i]),
    "blink_last_error": (_cp, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class BlinkError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"blink error {code} ({_lib.blink_result_string(code).decode()}): {msg}")
        self.code = code


def _check(code, comm=None):
    if code != 0:
        raise BlinkError(code, (_lib.blink_last_error(comm) or b"").decode())


def config(**kw):
    """blink_config_t with defaults (blink_config_default) overridden by kw."""
    c = _Config()
    _lib.blink_config_default(ctypes.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class Graph:
    """Link graph: nodes 0..nranks-1 are GPUs, then `switches` SWITCH
    nodes.  `links` = iterable of (src, dst, capacity, bidirectional)."""

    def __init__(self, nranks, links, switches=0):
        self.nranks = nranks
        n = nranks + switches
        self._kinds = (ctypes.c_int * n)(*([NODE_GPU] * nranks + [NODE_SWITCH] * switches))
        links = list(links)
        self._links = (_Link * max(1, len(links)))(*[_Link(int(a), int(b), float(c), int(d))
                                                       for a, b, c, d in links])
        self._g = _Graph(n, self._kinds, len(links), self._links)

    @classmethod
    def multi_server(cls, nranks, cap, servers, net_capacity=1.0):
        """NEXT-4: GPU-GPU links `cap` ({(u, v): c}) inside the servers plus one
        network SWITCH node (id nranks) linked to every GPU; links between
        servers are dropped.  `servers`: lists of ranks."""
        where = {v: i for i, s in enumerate(servers) for v in s}
        links = [(u, v, c, 0) for (u, v), c in sorted(cap.items()) if where[u] == where[v]]
        links += [(v, nranks, net_capacity, 1) for v in range(nranks)]
        return cls(nranks, links, switches=1)

    @classmethod
    def from_pairs(cls, nranks, cap):
        """From a directed capacity dict {(u, v): c} (the oracle's format)."""
        return cls(nranks, [(u, v, c, 0) for (u, v), c in sorted(cap.items())])

    def ptr(self):
        return ctypes.byref(self._g)


def miad(init=1 << 20, min_chunk=16 << 10, max_chunk=64 << 20):
    """A MIAD controller: returns (state, step) where step(throughput) -> next chunk."""
    st = Miad()
    _lib.blink_miad_init(ctypes.byref(st), init, min_chunk, max_chunk)
    return st, (lambda thr: _lib.blink_miad_step(ctypes.byref(st), float(thr)))


def _gptr(graph):
    return graph.ptr() if graph is not None else None


def _cptr(cfg):
    return ctypes.byref(cfg) if cfg is not None else None


def _json_call(fn, *args, comm=None):
    n = _sz(1 << 16)
    buf = ctypes.create_string_buffer(n.value)
    code = fn(*args, buf, ctypes.byref(n))
    if code != 0 and n.value > len(buf):
        buf = ctypes.create_string_buffer(n.value)
        code = fn(*args, buf, ctypes.byref(n))
    _check(code, comm)
    return json.loads(buf.value.decode())


def hybrid_split(d_total, bw_pcie, bw_nvl, t_dpa):
    """Eq. 8: (D_PCIe, D_NVL) bytes for the PCIe / NVLink trees."""
    a, b = _sz(), _sz()
    _check(_lib.blink_hybrid_split(d_total, bw_pcie, bw_nvl, t_dpa, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def topology_json(bus_ids):
    """Host-only topology probe of the GPUs with these PCI bus ids."""
    arr = (ctypes.c_char_p * len(bus_ids))(*[b.encode() for b in bus_ids])
    return _json_call(_lib.blink_topology_json, len(bus_ids), arr)


def plan_json(nranks, is_allreduce, root=0, count=0, dtype="f32", graph=None, cfg=None):
    """Host-only TreeGen + split/chunking for a graph (no GPU needed)."""
    return _json_call(_lib.blink_plan_json, _gptr(graph), nranks, _cptr(cfg), int(is_allreduce),
                      int(root), count, DTYPES[dtype])


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


_DT_CACHE = {}  # dtype object -> "f32" / "bf16" / "i32" (per-call cost: one dict lookup)


def _dtype_of(x, dtype):
    if dtype is not None:
        return dtype
    d = getattr(x, "dtype", None)
    v = _DT_CACHE.get(d)
    if v is not None:
        return v
    name = str(d)
    for k, v in (("float32", "f32"), ("bfloat16", "bf16"), ("int32", "i32")):
        if name.endswith(k):
            _DT_CACHE[d] = v
            return v
    raise ValueError(f"cannot infer dtype of {x!r}; pass dtype=")


_RAW_STREAM = []  # [fn(device) -> raw cudaStream_t int] once torch is loaded


def _stream(s, device=None):
    """The current torch stream of `device` (None: torch's current device) as
    a raw cudaStream_t.  torch's private raw-stream getter costs ~0.2 us per
    call against ~2.5 us for torch.cuda.current_stream(); the public API is
    the fallback."""
    if s is None:
        if _RAW_STREAM:
            return _RAW_STREAM[0](device)
        import sys
        torch = sys.modules.get("torch")
        if torch is None or not torch.cuda.is_available():
            return None
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            cur = torch.cuda.current_device
            _RAW_STREAM.append(lambda dev: raw(cur() if dev is None else dev))
        else:
            _RAW_STREAM.append(lambda dev: torch.cuda.current_stream(dev).cuda_stream)
        return _RAW_STREAM[0](device)
    if isinstance(s, int):
        return s
    return s.cuda_stream


class Comm:
    """One rank of a Blink communicator (a blink_comm_t)."""

    def __init__(self, handle):
        self._h = ctypes.c_void_p(handle)
        n, r, d = _i(), _i(), _i()
        _check(_lib.blink_comm_info(self._h, ctypes.byref(n), ctypes.byref(r), ctypes.byref(d)))
        self.nranks, self.rank, self.device = n.value, r.value, d.value

    def allreduce(self, send, recv=None, op="sum", count=None, dtype=None, stream=None):
        """AllReduce.  recv=None means in place."""
        recv = send if recv is None else recv
        dt = _dtype_of(send, dtype)
        cnt = send.numel() if count is None else count
        _check(_lib.blink_allreduce(self._h, _ptr(send), _ptr(recv), cnt, DTYPES[dt], OPS[op],
                                    _stream(stream, self.device)), self._h)
        return recv

    def broadcast(self, send, recv=None, root=0, count=None, dtype=None, stream=None):
        """Broadcast from `root`.  send is read on the root only."""
        recv = send if recv is None else recv
        ref = send if send is not None else recv
        dt = _dtype_of(ref, dtype)
        cnt = ref.numel() if count is None else count
        _check(_lib.blink_broadcast(self._h, _ptr(send), _ptr(recv), cnt, DTYPES[dt], int(root),
                                    _stream(stream, self.device)), self._h)
        return recv

    def reduce_scatter(self, send, recv, op="sum", recvcount=None, dtype=None, stream=None):
        """ReduceScatter (NEXT-3): send holds nranks blocks of recvcount; rank j
        receives block j reduced over all ranks."""
        dt = _dtype_of(recv, dtype)
        cnt = recv.numel() if recvcount is None else recvcount
        _check(_lib.blink_reduce_scatter(self._h, _ptr(send), _ptr(recv), cnt, DTYPES[dt], OPS[op],
                                         _stream(stream, self.device)), self._h)
        return recv

    def allgather(self, send, recv, sendcount=None, dtype=None, stream=None):
        """AllGather (NEXT-3): block `rank` of every recv gets this send."""
        dt = _dtype_of(send, dtype)
        cnt = send.numel() if sendcount is None else sendcount
        _check(_lib.blink_allgather(self._h, _ptr(send), _ptr(recv), cnt, DTYPES[dt],
                                    _stream(stream, self.device)), self._h)
        return recv

    def gather(self, send, recv=None, root=0, sendcount=None, dtype=None, stream=None):
        """Gather (NEXT-3): block `rank` of the root's recv gets this
        send; recv is ignored (may be None) on the other ranks."""
        dt = _dtype_of(send, dtype)
        cnt = send.numel() if sendcount is None else sendcount
        _check(_lib.blink_gather(self._h, _ptr(send), _ptr(recv), cnt, DTYPES[dt], int(root),
                                 _stream(stream, self.device)), self._h)
        return recv

    def plan(self, is_allreduce=True, root=0, count=0, dtype="f32"):
        return _json_call(_lib.blink_get_plan, self._h, int(is_allreduce), int(root), count,
                          DTYPES[dtype], comm=self._h)

    def stats(self):
        s = _Stats()
        _check(_lib.blink_get_stats(self._h, ctypes.byref(s)), self._h)
        return dict(launches=s.launches, last_ctas=s.last_ctas, last_chunks=s.last_chunks,
                    last_trees=s.last_trees, last_chunk_bytes=s.last_chunk_bytes,
                    last_steal_channels=s.last_steal_channels)

    def trace(self):
        """Per-CTA %globaltimer stamps of the last launch (BLINK_TRACE=1), as a
        list of 16-tuples (ns, include/blink.h blink_get_trace); empty when
        tracing is off."""
        n = _sz(0)
        _check(_lib.blink_get_trace(self._h, None, ctypes.byref(n)), self._h)
        if n.value == 0:
            return []
        buf = (ctypes.c_uint64 * n.value)()
        _check(_lib.blink_get_trace(self._h, buf, ctypes.byref(n)), self._h)
        return [tuple(buf[i:i + 16]) for i in range(0, n.value, 16)]

    def register(self, buf, nbytes, exchange):
        """Symmetric registration (multi-process).  `exchange(bytes) -> list[bytes]`
        all-gathers one blob per rank in rank order."""
        n = _sz(0)
        _check(_lib.blink_register_export(self._h, _ptr(buf), nbytes, None, ctypes.byref(n)), self._h)
        blob = ctypes.create_string_buffer(max(1, n.value))
        _check(_lib.blink_register_export(self._h, _ptr(buf), nbytes, blob, ctypes.byref(n)), self._h)
        blobs = exchange(blob.raw[:n.value])
        allb = b"".join(blobs)
        _check(_lib.blink_register_connect(self._h, _ptr(buf), allb, n.value), self._h)

    def destroy(self):
        if self._h:
            _check(_lib.blink_destroy(self._h))
            self._h = None


def init_all(devs, graph=None, cfg=None):
    """Single-process comms for ranks on `devs` (devices may repeat: virtual
    ranks sharing one GPU).  Collective calls are batched until every rank has
    called; then one launch per device runs."""
    n = len(devs)
    hs = (ctypes.c_void_p * n)()
    d = (ctypes.c_int * n)(*devs)
    _check(_lib.blink_init_all(hs, n, d, _gptr(graph), _cptr(cfg)))
    return [Comm(hs[i]) for i in range(n)]


def init_multiprocess(nranks, rank, device, exchange, graph=None, cfg=None):
    """One rank per process.  `exchange(bytes) -> list[bytes]` all-gathers the
    handle blobs (e.g. torch.distributed.all_gather_object over gloo)."""
    h = ctypes.c_void_p()
    _check(_lib.blink_init(ctypes.byref(h), nranks, rank, device, _gptr(graph), _cptr(cfg)))
    n = _sz(512)
    blob = ctypes.create_string_buffer(512)
    _check(_lib.blink_export_handle(h, blob, ctypes.byref(n)), h)
    blobs = exchange(blob.raw[:n.value])
    if len(blobs) != nranks or any(len(b) != n.value for b in blobs):
        raise BlinkError(5, "exchange returned the wrong number/size of blobs")
    _check(_lib.blink_connect(h, b"".join(blobs), n.value), h)
    return Comm(h.value)


def torch_exchange(group=None):
    """An `exchange` callable over torch.distributed (any backend)."""
    import torch.distributed as dist

    def ex(blob):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, blob, group=group)
        return out
    return ex
