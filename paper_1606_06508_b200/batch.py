"""Array plumbing between the public API and the C ABI.

Accepts ``[N, n]`` row arrays in either of two homes:

* a CUDA ``torch.Tensor`` -- outputs are allocated on the same device, the kernel is
  enqueued on torch's current stream of that device (``fn_run``), nothing synchronises;
* a host array (``numpy.ndarray`` or CPU ``torch.Tensor``) -- outputs are host arrays of
  the same kind; the library copies in, computes on the current CUDA device and copies
  out (``fn_host_run``: chunked H2D / kernel / D2H pipeline).  Page-locked (pinned)
  host memory gives full PCIe bandwidth.

Rows need not be dense: a view whose rows are ``ldx`` elements apart with unit column
stride (xyz of xyzw records, ``X[:, :n]`` of a wider array) runs as it is
(``fn_run_ld`` / ``fn_host_run_ld``); other layouts are gathered first.

No path computes on the CPU: without the CUDA library every call raises.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from typing import Any, NamedTuple

import numpy as np

from paper_1606_06508_b200 import _lib


class _Rows:
    """Default of the trailing components ``x2..xn`` in the public wrappers.  The
    reference's parameters (``normalize3(p, x1, x2, x3)``, normalize.py:58) keep their
    names and order; leaving ``x2..xn`` out is the batched overload, where ``x1`` is an
    ``[N, n]`` array of rows."""

    __slots__ = ()

    def __repr__(self) -> str:
        return "ROWS"


ROWS = _Rows()


def components(*xs) -> tuple:
    """The components a wrapper was called with (``x1`` alone for one row array)."""
    if xs[-1] is not ROWS:
        return xs
    return tuple(v for v in xs if v is not ROWS)


def widths(op: int, dim: int) -> tuple[int, int, int]:
    """Elements per row of the (head, body, extra) outputs of a kernel family."""
    if op == _lib.OP_NORM:
        return 1, 0, 0
    if op == _lib.OP_NORMALIZE_SQ:
        return 1, dim, 1
    if op in (_lib.OP_ROT_UNIT, _lib.OP_ROT_GENERAL):
        return 9, 0, 0
    if op == _lib.OP_NORMALIZE_ROT:
        return 1, 4, 9
    if op == _lib.OP_ROT_APPLY:
        return 3, 0, 0
    return 1, dim, 0


def _shape(n: int, w: int) -> tuple[int, ...]:
    return (n,) if w == 1 else ((n, 3, 3) if w == 9 else (n, w))


_host = threading.local()


@contextmanager
def host_devices(devices):
    """Within the scope (this thread), host-array calls -- ``[N, n]`` rows and component
    arrays alike -- shard their rows over ``devices`` (CUDA ordinals), one host thread
    per device (fn_host_run_multi / fn_host_run_soa_multi)."""
    devs = [int(d) for d in devices]
    if not devs:
        raise ValueError("host_devices needs at least one device")
    prev = getattr(_host, "devices", None)
    _host.devices = devs
    try:
        yield devs
    finally:
        _host.devices = prev


def host_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised numpy array in page-locked (portable) host memory from
    ``fn_host_alloc``.  Host-array calls DMA such buffers directly instead of staging
    them (1.56 vs 0.64 Gvec/s for 3-D f64 rows with inputs and outputs page-locked).
    The memory is released (``fn_host_free``) when the array and every view of it are
    gone.  Allocation pins pages, so reuse these buffers across calls."""
    import ctypes
    import weakref

    shape = (int(shape),) if np.isscalar(shape) else tuple(int(d) for d in shape)
    dt = np.dtype(dtype)
    count = int(np.prod(shape, dtype=np.int64))
    nbytes = count * dt.itemsize
    if nbytes == 0:
        return np.empty(shape, dtype=dt)
    L = _lib.lib()
    ptr = ctypes.c_void_p()
    _lib.check(L.fn_host_alloc(nbytes, ctypes.byref(ptr)), "fn_host_alloc")
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    weakref.finalize(buf, L.fn_host_free, ptr.value)
    return np.frombuffer(buf, dtype=dt, count=count).reshape(shape)


class _PinnedPool:
    """Page-locked blocks for the outputs of host-array calls made without ``out=``.

    Results the library allocates itself land in page-locked memory, so the D2H copies
    go straight into them: no staging copy, no first-touch page faults in a fresh
    ``np.empty``.  Pinning is slow (``cudaHostAlloc`` zeroes and locks every page), so
    blocks are recycled: when a result array and all its views are gone, its block goes
    back to a free list by size class (sizes rounded up by at most 1/8), and the next
    call of that size class reuses it.  The free lists hold at most
    FASTNORM_B200_HOST_POOL_MB (default: a quarter of the host's memory); beyond that,
    blocks are released.  FASTNORM_B200_HOST_POOL_MB=0 turns the pool off (plain
    ``np.empty`` outputs, staged on the way back)."""

    MIN_BYTES = 128 << 10  # smaller outputs take the zero-copy small-batch route anyway

    def __init__(self):
        self._lock = threading.Lock()
        self._free: dict[int, list[int]] = {}
        self._cached = 0
        self._limit: int | None = None
        self.allocs = 0  # blocks pinned so far (fn_host_alloc calls)
        self.reuses = 0

    def limit(self) -> int:
        if self._limit is None:
            import os

            env = os.environ.get("FASTNORM_B200_HOST_POOL_MB")
            if env is not None:
                self._limit = max(0, int(env)) << 20
            else:
                try:
                    self._limit = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") // 4
                except (ValueError, OSError):
                    self._limit = 8 << 30
        return self._limit

    @staticmethod
    def size_class(nbytes: int) -> int:
        step = max(64 << 10, 1 << max(0, nbytes.bit_length() - 4))
        return -(-nbytes // step) * step

    def empty(self, shape, dtype: np.dtype) -> np.ndarray:
        import ctypes
        import weakref

        count = 1
        for d in shape:
            count *= d
        nbytes = count * dtype.itemsize
        if nbytes < self.MIN_BYTES or self.limit() == 0:
            return np.empty(shape, dtype=dtype)
        cls = self.size_class(nbytes)
        ptr = None
        with self._lock:
            lst = self._free.get(cls)
            if lst:
                ptr = lst.pop()
                self._cached -= cls
                self.reuses += 1
        if ptr is None:
            L = _lib.lib()
            p = ctypes.c_void_p()
            if L.fn_host_alloc(cls, ctypes.byref(p)) != 0:
                return np.empty(shape, dtype=dtype)  # cannot pin more: a pageable result
            ptr = p.value
            with self._lock:
                self.allocs += 1
        buf = (ctypes.c_char * cls).from_address(ptr)
        fin = weakref.finalize(buf, self._give, ptr, cls)
        fin.atexit = False  # at exit the process releases everything anyway
        return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)

    def _give(self, ptr: int, cls: int) -> None:
        with self._lock:
            if self._cached + cls <= self.limit():
                self._free.setdefault(cls, []).append(ptr)
                self._cached += cls
                return
        _lib.lib().fn_host_free(ptr)

    def clear(self) -> None:
        """Release every cached block (results still alive keep theirs)."""
        with self._lock:
            blocks = [p for lst in self._free.values() for p in lst]
            self._free.clear()
            self._cached = 0
        for ptr in blocks:
            _lib.lib().fn_host_free(ptr)


pinned_pool = _PinnedPool()


class BatchOut(NamedTuple):
    head: Any
    body: Any
    sq: Any


def _torch():
    import torch  # local: the numpy path must not pay for importing torch

    return torch


_torch_types: set = set()  # tensor classes seen so far (the check runs several times per call)


def is_torch(x) -> bool:
    t = type(x)
    if t in _torch_types:
        return True
    if t is np.ndarray:
        return False
    if t.__module__.startswith("torch") and t.__name__ in ("Tensor", "Parameter"):
        _torch_types.add(t)
        return True
    return False


def is_array(x) -> bool:
    """True for the batched overloads (an ``[N, n]`` array instead of n scalars)."""
    return isinstance(x, np.ndarray) or is_torch(x)


def _dtype_code(dtype_name: str) -> int:
    if dtype_name == "float64":
        return _lib.F64
    if dtype_name == "float32":
        return _lib.F32
    raise TypeError(f"rows must be float32 or float64, got {dtype_name}")


_prec_of: dict = {}


def precision_of(x) -> str:
    dt = x.dtype
    prec = _prec_of.get(dt)
    if prec is None:
        name = str(dt).replace("torch.", "")
        prec = _prec_of[dt] = "double" if _dtype_code(name) == _lib.F64 else "single"
    return prec


def _check_out(o, shape, like, what):
    if o is None:
        return None
    if type(o) is np.ndarray and type(like) is np.ndarray:
        if o.dtype == like.dtype and o.shape == shape and o.flags.c_contiguous:
            return o  # the common host case
    elif (is_torch(like) and is_torch(o) and o.dtype == like.dtype and o.shape == shape
            and o.device == like.device and o.is_contiguous()):
        return o  # the common case, without building messages or dtype strings
    if tuple(o.shape) != tuple(shape):
        raise ValueError(f"out {what} has shape {tuple(o.shape)}, expected {tuple(shape)}")
    if str(o.dtype) != str(like.dtype):
        raise TypeError(f"out {what} has dtype {o.dtype}, expected {like.dtype}")
    if is_torch(like):
        if not is_torch(o) or o.device != like.device or not o.is_contiguous():
            raise ValueError(f"out {what} must be a contiguous tensor on {like.device}")
    elif not (isinstance(o, np.ndarray) and o.flags.c_contiguous):
        raise ValueError(f"out {what} must be a C-contiguous numpy array")
    return o


_fast: list = []


def _fast_run():
    """fn_run through the CPython extension (csrc/scalar_ext.c), or None if not built."""
    if not _fast:
        import ctypes

        try:
            from paper_1606_06508_b200 import _scalar
        except ImportError:
            _fast.append(None)
        else:
            L = _lib.lib()
            _scalar.bind_run(ctypes.cast(L.fn_run, ctypes.c_void_p).value)
            _scalar.bind_host(ctypes.cast(L.fn_host_run, ctypes.c_void_p).value)
            _fast.append(_scalar)
    return _fast[0]


_ka_addrs: dict = {}


def _ka_address(ka_arr: np.ndarray) -> int:
    """Address of a kernel-argument array; read-only arrays (kernel_args_array's cached
    ones) are remembered together with a reference, so the address stays valid."""
    if ka_arr.flags.writeable:
        return ka_arr.ctypes.data
    hit = _ka_addrs.get(id(ka_arr))
    if hit is None or hit[0] is not ka_arr:
        hit = _ka_addrs[id(ka_arr)] = (ka_arr, ka_arr.ctypes.data)
    return hit[1]


_stream_of = None
_device_of = None
_dcode_of: dict = {}


def _current_device(torch) -> int:
    """torch's current CUDA device (the cheap private accessor when present)."""
    global _device_of
    if _device_of is None:
        _device_of = getattr(torch._C, "_cuda_getDevice", None) or torch.cuda.current_device
    return _device_of()


def _cuda_stream(torch, dev: int) -> int:
    """torch's current stream on device ``dev`` as a raw handle (the cheap private
    accessor when present)."""
    global _stream_of
    if _stream_of is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        _stream_of = raw if raw is not None else (lambda d: torch.cuda.current_stream(d).cuda_stream)
    return _stream_of(dev)


def _overlaps(x, n: int, ldx: int, dim: int, outs) -> bool:
    """Whether any output tensor's bytes meet the span of strided rows x."""
    es = x.element_size()
    lo = x.data_ptr()
    hi = lo + ((n - 1) * ldx + dim) * es
    for o in outs:
        if o is not None and o.numel():
            a = o.data_ptr()
            if a < hi and lo < a + o.numel() * es:
                return True
    return False


def _run_device_out(op, dim, x, n, ka_arr, out, w0, w1, w2):
    """The common device call -- dense CUDA rows on torch's current device, valid
    preallocated outputs, a non-rotation op -- with no further checks; None when any
    condition fails (the general path then handles the call, including its errors)."""
    fast = _fast_run()
    if fast is None or not x.is_cuda or not x.is_contiguous() or op > _lib.OP_NORMALIZE_SQ:
        return None
    dt, dev = x.dtype, x.device
    outs = tuple(out)
    if len(outs) != 1 + (w1 > 0) + (w2 > 0):
        return None
    for o, w in zip(outs, (w0,) + ((w1,) if w1 else ()) + ((w2,) if w2 else ())):
        if type(o) not in _torch_types or o.dtype is not dt or o.device != dev or not o.is_contiguous() \
                or o.shape != _shape(n, w):
            return None
    torch = _torch()
    if _current_device(torch) != dev.index:
        return None
    dcode = _dcode_of.get(dt)
    if dcode is None:
        return None
    head, body, extra = outs[0], outs[1] if w1 else None, outs[-1] if w2 else None
    rc = fast.run(op, dim, dcode, x.data_ptr(), n, head.data_ptr(), None if body is None else body.data_ptr(),
                  None if extra is None else extra.data_ptr(), None if ka_arr is None else _ka_address(ka_arr),
                  _cuda_stream(torch, dev.index))
    if rc:
        _lib.check(rc, "fn_run")
    return BatchOut(head, body, extra)


def run(op: int, dim: int, x, ka_arr: np.ndarray | None, out=None, invalid=None) -> BatchOut:
    """Run kernel family ``op`` over rows ``x[N, dim]``; return (head, body, extra).

    ``invalid`` (device path, rotations): a CUDA int64 tensor the kernel adds the number
    of rejected rows to."""
    if x.ndim != 2 or x.shape[1] != dim:
        raise ValueError(f"expected rows of shape [N, {dim}], got {tuple(x.shape)}")
    w0, w1, w2 = widths(op, dim)
    n = int(x.shape[0])
    if out is not None and invalid is None and type(x) in _torch_types:
        res = _run_device_out(op, dim, x, n, ka_arr, out, w0, w1, w2)
        if res is not None:
            return res
    L = _lib.lib()
    kptr = None if ka_arr is None else _ka_address(ka_arr)
    outs = tuple(out) if out is not None else ()
    want = 1 + int(w1 > 0) + int(w2 > 0)
    if out is not None and len(outs) != want:
        raise ValueError(f"out must hold {want} arrays")
    o_head = outs[0] if outs else None
    o_body = outs[1] if outs and w1 else None
    o_extra = outs[-1] if outs and w2 else None

    if is_torch(x):
        torch = _torch()
        dcode = _dcode_of.get(x.dtype)
        if dcode is None:
            dcode = _dcode_of[x.dtype] = _dtype_code(str(x.dtype).replace("torch.", ""))
        if x.is_cuda:
            # Rows that are ldx elements apart (padded records, X[:, :dim] of a wider
            # array) go to fn_run_ld as they are; any other layout is gathered first.
            ldx = dim
            rot = op in (_lib.OP_ROT_UNIT, _lib.OP_ROT_GENERAL, _lib.OP_NORMALIZE_ROT)
            if not x.is_contiguous():
                if not rot and x.stride(1) == 1 and x.stride(0) >= dim and n > 0:
                    ldx = int(x.stride(0))
                else:
                    x = x.contiguous()

            def alloc(o, w, what):
                if not w:
                    return None
                o = _check_out(o, _shape(n, w), x, what)
                return o if o is not None else x.new_empty(_shape(n, w))

            head, body, extra = alloc(o_head, w0, "head"), alloc(o_body, w1, "body"), alloc(o_extra, w2, "extra")
            if ldx != dim and _overlaps(x, n, ldx, dim, (head, body, extra)):
                # an output written over strided input rows of other tiles: gather first
                x, ldx = x.contiguous(), dim
            ptr = (lambda t: None if t is None else t.data_ptr())
            dev = x.device.index
            # The library launches on the thread's current CUDA device (shared with torch
            # through the driver's current context): switch only when x lives elsewhere.
            switch = _current_device(torch) != dev
            if switch:
                ctx = torch.cuda.device(dev)
                ctx.__enter__()
            try:
                stream = _cuda_stream(torch, dev)
                if rot:
                    rc = L.fn_run_rot(op, x.data_ptr(), n, ptr(head), ptr(body), ptr(extra), kptr,
                                      ptr(invalid), stream)
                elif ldx != dim:
                    rc = L.fn_run_ld(op, dim, dcode, x.data_ptr(), n, ldx, ptr(head), ptr(body), ptr(extra),
                                     kptr, stream)
                else:
                    fast = _fast_run()
                    call = fast.run if fast is not None else L.fn_run
                    rc = call(op, dim, dcode, x.data_ptr(), n, ptr(head), ptr(body), ptr(extra), kptr, stream)
            finally:
                if switch:
                    ctx.__exit__(None, None, None)
            if rc:
                _lib.check(rc, "fn_run")
            return BatchOut(head, body, extra)
        # CPU tensor: host path, results as CPU tensors sharing the numpy buffers
        res = run(op, dim, x.numpy(), ka_arr,
                  None if out is None else tuple(o.numpy() for o in outs))
        conv = (lambda a: None if a is None else torch.from_numpy(a))
        return BatchOut(conv(res.head), conv(res.body), conv(res.sq))

    if not isinstance(x, np.ndarray):
        raise TypeError(f"rows must be a numpy array or torch tensor, got {type(x).__name__}")
    dcode = _dcode_of.get(x.dtype)
    if dcode is None:
        dcode = _dcode_of[x.dtype] = _dtype_code(str(x.dtype))
    # Rows ldx elements apart (padded records, X[:, :dim] of a wider array) cross PCIe as
    # they are (fn_host_run_ld); any other layout is gathered first.
    ldx = dim
    if not x.flags.c_contiguous:
        es = x.itemsize
        st0, st1 = x.strides
        rot = op in (_lib.OP_ROT_UNIT, _lib.OP_ROT_GENERAL, _lib.OP_NORMALIZE_ROT)
        if not rot and n > 0 and st1 == es and st0 % es == 0 and st0 >= dim * es:
            ldx = st0 // es
        else:
            x = np.ascontiguousarray(x)

    def alloc_np(o, w, what):
        if not w:
            return None
        o = _check_out(o, _shape(n, w), x, what)
        return o if o is not None else pinned_pool.empty(_shape(n, w), x.dtype)

    head, body, extra = alloc_np(o_head, w0, "head"), alloc_np(o_body, w1, "body"), alloc_np(o_extra, w2, "extra")
    if ldx != dim and any(o is not None and np.may_share_memory(x, o) for o in (head, body, extra)):
        x, ldx = np.ascontiguousarray(x), dim  # outputs written over strided input rows
    ptr = (lambda a: None if a is None else a.ctypes.data)
    devs = getattr(_host, "devices", None)
    if devs:
        darr = np.array(devs, dtype=np.int32)
        rc = L.fn_host_run_multi_ld(op, dim, dcode, x.ctypes.data, n, ldx, ptr(head), ptr(body), ptr(extra),
                                    kptr, darr.ctypes.data, len(devs))
        _lib.check(rc, "fn_host_run_multi")
    elif ldx != dim:
        rc = L.fn_host_run_ld(op, dim, dcode, x.ctypes.data, n, ldx, ptr(head), ptr(body), ptr(extra), kptr)
        _lib.check(rc, "fn_host_run")
    else:
        fast = _fast_run()
        if fast is not None:
            rc = fast.host_run(op, dim, dcode, x, n, head, body, extra, kptr)
        else:
            rc = L.fn_host_run(op, dim, dcode, x.ctypes.data, n, ptr(head), ptr(body), ptr(extra), kptr)
        if rc:
            _lib.check(rc, "fn_host_run")
    return BatchOut(head, body, extra)


def run_many(op: int, dim: int, xs, ka_arr: np.ndarray | None, outs=None) -> list:
    """Kernel family ``op`` over several independent ``[N_j, dim]`` row arrays; returns
    one BatchOut per array.  CUDA tensors (one device, one dtype) go to the device in one
    launch per 48 arrays (fn_run_many); host arrays are run one by one (fn_host_run).
    ``outs``: optional list of per-array ``out`` tuples, as for ``run``."""
    import ctypes

    xs = list(xs)
    if outs is not None and len(outs) != len(xs):
        raise ValueError("outs must hold one entry per array")
    if not xs:
        return []
    if not all(is_torch(x) and x.is_cuda for x in xs):
        return [run(op, dim, x, ka_arr, None if outs is None else outs[j]) for j, x in enumerate(xs)]
    torch = _torch()
    dev, dt = xs[0].device, xs[0].dtype
    if any(x.device != dev or x.dtype != dt for x in xs):
        raise TypeError("arrays must share device and dtype")
    for x in xs:
        if x.ndim != 2 or x.shape[1] != dim:
            raise ValueError(f"expected rows of shape [N, {dim}], got {tuple(x.shape)}")
    xs = [x if x.is_contiguous() else x.contiguous() for x in xs]
    dcode = _dcode_of.get(dt)
    if dcode is None:
        dcode = _dcode_of[dt] = _dtype_code(str(dt).replace("torch.", ""))
    w0, w1, w2 = widths(op, dim)
    kinds = [(w0, "head")] + ([(w1, "body")] if w1 else []) + ([(w2, "extra")] if w2 else [])
    res = []
    for j, x in enumerate(xs):
        o = outs[j] if outs is not None and outs[j] is not None else ()
        n = x.shape[0]
        arrays = []
        for k, (w, what) in enumerate(kinds):
            shape = _shape(n, w)
            t = o[k] if len(o) > k else None
            if t is None:
                t = x.new_empty(shape)
            elif not (t.dtype is dt and t.device == dev and t.shape == shape and t.is_contiguous()):
                t = _check_out(t, shape, x, what)
            arrays.append(t)
        res.append(BatchOut(arrays[0], arrays[1] if w1 else None, arrays[-1] if w2 else None))
    m = len(xs)
    arr = (lambda vals: (ctypes.c_void_p * m)(*vals))
    xp = arr([x.data_ptr() for x in xs])
    hp = arr([r.head.data_ptr() for r in res])
    bp = arr([r.body.data_ptr() for r in res]) if w1 else None
    qp = arr([r.sq.data_ptr() for r in res]) if w2 else None
    ns = (ctypes.c_int64 * m)(*[int(x.shape[0]) for x in xs])
    kptr = None if ka_arr is None else _ka_address(ka_arr)
    with torch.cuda.device(dev):
        rc = _lib.lib().fn_run_many(op, dim, dcode, m, ctypes.addressof(xp), ctypes.addressof(ns),
                                    ctypes.addressof(hp), None if bp is None else ctypes.addressof(bp),
                                    None if qp is None else ctypes.addressof(qp), kptr,
                                    _cuda_stream(torch, dev.index))
    if rc:
        _lib.check(rc, "fn_run_many")
    return res


def run_rows2(op: int, a, v, ka_arr: np.ndarray | None, out=None, invalid=None):
    """Two-input ops (per-row rotation of vectors): a = q[N, 4] (OP_QUAT_ROTATE) or
    R[N, 9] (OP_MAT_APPLY), v[N, 3], both float64 and in the same home (CUDA tensors on
    one device, or host arrays).  Returns out[N, 3] of the same kind.

    ``invalid`` (device path): a CUDA int64 tensor the kernel adds rejected rows to."""
    width = 4 if op == _lib.OP_QUAT_ROTATE else 9
    n = int(v.shape[0])
    if tuple(v.shape) != (n, 3):
        raise ValueError(f"vectors must have shape [N, 3], got {tuple(v.shape)}")
    if tuple(a.shape) != (n, width):
        raise ValueError(f"expected [{n}, {width}] records for the rotations, got {tuple(a.shape)}")
    for t, what in ((a, "rotations"), (v, "vectors")):
        if str(t.dtype).replace("torch.", "") != "float64":
            raise TypeError(f"{what} must be float64 (the reference computes in double)")
    L = _lib.lib()
    kptr = None if ka_arr is None else ka_arr.ctypes.data
    if is_torch(a) and a.is_cuda:
        torch = _torch()
        if not (is_torch(v) and v.is_cuda and v.device == a.device):
            raise ValueError("rotations and vectors must be CUDA tensors on the same device")
        a, v = a.contiguous(), v.contiguous()
        o = _check_out(out, (n, 3), v, "out") if out is not None else torch.empty((n, 3), dtype=v.dtype, device=v.device)
        with torch.cuda.device(v.device):
            rc = L.fn_rotate_rows_f64(op, a.data_ptr(), v.data_ptr(), n, o.data_ptr(), kptr,
                                      None if invalid is None else invalid.data_ptr(),
                                      torch.cuda.current_stream(v.device).cuda_stream)
        _lib.check(rc, "fn_rotate_rows_f64")
        return o
    if is_torch(a) or is_torch(v):
        res = run_rows2(op, np.asarray(a.numpy() if is_torch(a) else a), np.asarray(v.numpy() if is_torch(v) else v),
                        ka_arr, None if out is None else np.asarray(out.numpy() if is_torch(out) else out))
        return _torch().from_numpy(res) if is_torch(v) else res
    a, v = np.ascontiguousarray(a), np.ascontiguousarray(v)
    o = _check_out(out, (n, 3), v, "out") if out is not None else pinned_pool.empty((n, 3), np.dtype(np.float64))
    rc = L.fn_host_rotate_rows_f64(op, a.ctypes.data, v.ctypes.data, n, o.ctypes.data, kptr)
    _lib.check(rc, "fn_host_rotate_rows_f64")
    return o


def is_soa(xs, dim: int) -> bool:
    """The reference's scalar signature called with one 1-D array per component."""
    return len(xs) == dim and all(is_array(v) and v.ndim == 1 for v in xs)


def _columns_of_records(xs, dim: int):
    """If the component arrays are consecutive columns of one array of records (same
    dtype and home, one common row stride >= dim elements, column k starting k elements
    after column 0), return that [N, dim] strided view of the records, else None."""
    x0 = xs[0]
    if is_torch(x0):
        if not all(is_torch(v) and v.dim() == 1 and v.dtype == x0.dtype and v.device == x0.device for v in xs):
            return None
        es, st = x0.element_size(), x0.stride(0)
        if len(x0) < 2 or st < dim or any(v.stride(0) != st for v in xs):
            return None
        if any(v.data_ptr() != x0.data_ptr() + k * es for k, v in enumerate(xs)):
            return None
        return x0.as_strided((len(x0), dim), (st, 1))
    if not all(isinstance(v, np.ndarray) and v.ndim == 1 and v.dtype == x0.dtype for v in xs):
        return None
    es, st = x0.itemsize, x0.strides[0]
    if len(x0) < 2 or st % es or st < dim * es or any(v.strides[0] != st for v in xs):
        return None
    if any(v.ctypes.data != x0.ctypes.data + k * es for k, v in enumerate(xs)):
        return None
    return np.lib.stride_tricks.as_strided(x0, shape=(len(x0), dim), strides=(st, es), writeable=False)


def _run_soa_host(op: int, dim: int, xs, ka_arr: np.ndarray | None):
    """Host component arrays (numpy or CPU tensors) through fn_host_run_soa: the chunked
    host pipeline, no torch transfers.  Outputs are arrays of the inputs' kind."""
    import ctypes

    as_tensor = is_torch(xs[0])
    arrs = [np.ascontiguousarray(v.numpy() if is_torch(v) else np.asarray(v)) for v in xs]
    n = arrs[0].shape[0]
    dt = arrs[0].dtype
    if any(a.dtype != dt or a.ndim != 1 for a in arrs):
        raise TypeError("component arrays must be 1-D and share a dtype")
    dcode = _dtype_code(str(dt))
    w0, w1, w2 = widths(op, dim)
    head = pinned_pool.empty((n,), dt)
    body = [pinned_pool.empty((n,), dt) for _ in range(dim)] if w1 else None
    extra = pinned_pool.empty((n,), dt) if w2 else None
    xp = (ctypes.c_void_p * dim)(*[a.ctypes.data for a in arrs])
    bp = (ctypes.c_void_p * dim)(*[b.ctypes.data for b in body]) if body else None
    kptr = None if ka_arr is None else _ka_address(ka_arr)
    bptr = None if bp is None else ctypes.addressof(bp)
    eptr = None if extra is None else extra.ctypes.data
    devs = getattr(_host, "devices", None)
    if devs:  # shard over the scoped devices, as the AoS host calls do
        darr = np.array(devs, dtype=np.int32)
        rc = _lib.lib().fn_host_run_soa_multi(op, dim, dcode, ctypes.addressof(xp), n, head.ctypes.data, bptr,
                                              eptr, kptr, darr.ctypes.data, len(devs))
    else:
        rc = _lib.lib().fn_host_run_soa(op, dim, dcode, ctypes.addressof(xp), n, head.ctypes.data, bptr, eptr,
                                        kptr)
    if rc:
        _lib.check(rc, "fn_host_run_soa")
    if as_tensor:
        torch = _torch()
        conv = torch.from_numpy
        return conv(head), None if body is None else tuple(conv(b) for b in body), \
            None if extra is None else conv(extra)
    return head, None if body is None else tuple(body), extra


def run_soa(op: int, dim: int, xs, ka_arr: np.ndarray | None):
    """Structure-of-arrays rows: component arrays xs[k][N] -> (head[N], body tuple of
    dim arrays or None, extra[N] or None), through fn_run_soa on the device.

    CUDA tensors are used in place.  Host arrays (numpy, CPU tensors) go through the
    host pipeline (fn_host_run_soa).  Consecutive columns of one record array run the
    AoS kernels on the records in place."""
    import ctypes

    n = int(xs[0].shape[0])
    if any(int(v.shape[0]) != n for v in xs):
        raise ValueError("component arrays must have the same length")
    aos = _columns_of_records(xs, dim)
    if aos is not None:
        # the components are the columns of one record array (X[:, 0], X[:, 1], ...):
        # run the AoS kernels on the records in place, return column views
        res = run(op, dim, aos, ka_arr)
        body = None if res.body is None else tuple(res.body[:, k] for k in range(dim))
        return res.head, body, res.sq
    if not (is_torch(xs[0]) and xs[0].is_cuda):
        return _run_soa_host(op, dim, xs, ka_arr)
    torch = _torch()
    ts = [v.contiguous() for v in xs]
    dev = ts[0].device
    dt = ts[0].dtype
    if any(t.dtype != dt or t.device != dev for t in ts):
        raise TypeError("component arrays must share dtype and device")
    dcode = _dtype_code(str(dt).replace("torch.", ""))
    w0, w1, w2 = widths(op, dim)
    head = torch.empty(n, dtype=dt, device=dev)
    body = [torch.empty(n, dtype=dt, device=dev) for _ in range(dim)] if w1 else None
    extra = torch.empty(n, dtype=dt, device=dev) if w2 else None
    xp = (ctypes.c_void_p * dim)(*[t.data_ptr() for t in ts])
    bp = (ctypes.c_void_p * dim)(*[t.data_ptr() for t in body]) if body else None
    kptr = None if ka_arr is None else _ka_address(ka_arr)
    with torch.cuda.device(dev):
        rc = _lib.lib().fn_run_soa(op, dim, dcode, ctypes.addressof(xp), n, head.data_ptr(),
                                   None if bp is None else ctypes.addressof(bp),
                                   None if extra is None else extra.data_ptr(), kptr,
                                   _cuda_stream(torch, dev.index))
    if rc:
        _lib.check(rc, "fn_run_soa")
    return head, None if body is None else tuple(body), extra
