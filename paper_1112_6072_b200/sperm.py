"""Thin ctypes binding of libsperm.so (include/sperm.h), same names as the C ABI.

Argument marshalling only: torch CUDA tensors are passed as raw device pointers
together with torch's current CUDA stream; every step of the method runs in the
library's sm_100a kernels (or, for the scheduler and CRT, in its host C++ code).
There is NO fallback: if libsperm.so is missing or a call fails, an exception
is raised.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPERM_LIB: an alternative in-tree build of the library (A-B variants, tools/build_variant.py)
LIB_PATH = os.environ.get("SPERM_LIB") or os.path.join(_HERE, "libsperm.so")

KMAX = 8
NMAX = 48
EXPAND_NMAX = 128

OK, ERR_ARG, ERR_CUDA, ERR_RANGE, ERR_CAPACITY, ERR_PRIMES = 0, -1, -2, -3, -4, -5


class SpermError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libsperm error {code}: {msg}")
        self.code = code


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int

_SIGS = {
    "sperm_version": (_I, []),
    "sperm_last_error": (ctypes.c_char_p, []),
    "sperm_prime": (ctypes.c_uint32, [_I]),
    "sperm_crt": (_I, [_P, _I, _P, _I, _P]),
    "sperm_crt_batch": (_I, [_P, _I64, _I, _P, _I, _P, _I, _P]),
    "sperm_crt_device": (_I, [_P, _I64, _I, _P, _I, _P, _I, _P]),
    "sperm_bound_primes": (_I, [_P, _I, _P]),
    "sperm_permanent": (_I, [_P, _I, _I64, _P, _P, _P, _I64, _I, _I, _P, _P, _P, _P, _P]),
    "sperm_permanent_host": (_I, [_P, _I, _I64, _I, _P, _I, _P]),
    "sperm_rnw_terms": (ctypes.c_double, [_I, _I64]),
    "sperm_rnw_stats": (_I, [_P, _P, _P, _I]),
    "sperm_reduce_mod": (_I, [_P, _I64, _P, _P]),
    "sperm_fold_mod": (_I, [_P, _I64, _P]),
    "sperm_expand": (_I, [_P, _P, _P, _I, _I64, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    "sperm_expand_unordered": (_I, [_P, _P, _P, _I, _I64, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    "sperm_expand_stats": (_I, [_P, _P, _I]),
    "sperm_expand_subtree": (_I, [_P, _P, _P, _I, _I64, _I, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    "sperm_expand_subtree_stats": (_I, [_P, _P, _I]),
    "sperm_nnz": (_I, [_P, _I, _I64, _P, _P]),
    "sperm_estimate": (_I, [_P, _I, _I64, _P, _I, ctypes.c_uint64, _P, _P, _P]),
    "sperm_estimate_stats": (_I, [_P, _P, _I]),
    "sperm_schedule": (_I, [_P, _I64, _I, _I, ctypes.c_uint64, _P, _P, _P]),
    "sperm_kendall_tau": (_I, [_P, _P, _I64, _P, _P]),
    "sperm_list_schedule": (_I, [_P, _P, _I64, _I, _P, _P]),
    "sperm_interpolate_mod": (_I, [_P, _I, _P, _I, _I, _P, _I]),
    "sperm_queue_create": (_I, [_P, _P]),
    "sperm_queue_open": (_I, [_P, _P]),
    "sperm_queue_claim": (_I, [_P, _I64, _P, _P, _P]),
    "sperm_queue_close": (_I, [_P, _I]),
    "sperm_launch_count": (_I64, [_I]),
    "sperm_timing_enable": (None, [_I]),
    "sperm_timing_reset": (None, []),
    "sperm_timing_get": (_I, [ctypes.c_char_p, _P, _P]),
}
SYMBOLS = tuple(_SIGS)


def lib():
    """Load libsperm.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1112_6072_b200.build` "
                              "or __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise SpermError(rc, lib().sperm_last_error().decode())


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream=None) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _dev(t, dtype):
    """Require a contiguous CUDA tensor of the given dtype (no silent host copies)."""
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"expected dtype {dtype}, got {t.dtype}")
    return t.contiguous()


# --------------------------------------------------------------------- utility
def sperm_version() -> int:
    return lib().sperm_version()


def sperm_prime(i: int) -> int:
    return int(lib().sperm_prime(i))


def primes(k: int = KMAX) -> List[int]:
    return [sperm_prime(i) for i in range(k)]


def sperm_crt(residues: Sequence[int], k: int) -> int:
    """Host CRT (Garner) of residues[:k] to the symmetric-range integer."""
    r = np.ascontiguousarray(np.asarray(residues[:k], dtype=np.uint32))
    limbs = k + 2
    mag = np.zeros(limbs, dtype=np.uint32)
    sign = ctypes.c_int(0)
    _check(lib().sperm_crt(r.ctypes.data, k, mag.ctypes.data, limbs, ctypes.byref(sign)))
    v = 0
    for w in mag[::-1]:
        v = (v << 32) | int(w)
    return sign.value * v


def sperm_bound_primes(a) -> int:
    """CRT primes that reconstruct per(A) of a host matrix (row/col sums, Bregman-Minc)."""
    m = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    k = ctypes.c_int(0)
    _check(lib().sperm_bound_primes(m.ctypes.data if m.size else None, int(m.shape[0]) if m.ndim == 2 else 0,
                                    ctypes.byref(k)))
    return k.value


# --------------------------------------------------------------------- R-NW
def sperm_permanent(mats, coef=None, order=None, job=None, num_jobs: int = 0, min_primes: int = 1,
                    max_primes: int = 0, leaf_res=None, leaf_k=None, job_acc=None, leaf_cycles=None,
                    stream=None):
    """Batched R-NW leaf permanents mod the CRT primes (see include/sperm.h).

    mats: int32 CUDA tensor [count, n, n].  Outputs are allocated if not given:
    returns (leaf_res uint32-as-int32 [count, KMAX], leaf_k int32 [count])."""
    import torch
    mats = _dev(mats, torch.int32)
    count, n = int(mats.shape[0]), int(mats.shape[1]) if mats.dim() == 3 else 0
    dev = mats.device
    if leaf_res is None:
        leaf_res = torch.empty((count, KMAX), dtype=torch.int32, device=dev)
    if leaf_k is None:
        leaf_k = torch.empty((count,), dtype=torch.int32, device=dev)
    coef = _dev(coef, torch.int64)
    order = _dev(order, torch.int32)
    job = _dev(job, torch.int32)
    _check(lib().sperm_permanent(_ptr(mats), n, count, _ptr(coef), _ptr(order), _ptr(job), int(num_jobs),
                                 int(min_primes), int(max_primes), _ptr(leaf_res), _ptr(leaf_k), _ptr(job_acc),
                                 _ptr(leaf_cycles), _stream(stream)))
    return leaf_res, leaf_k


def sperm_permanent_host(h_mats, min_primes: int = 1, out=None, stream=None) -> List[int]:
    """Exact permanents of a HOST batch [count, n, n] int32 (numpy, ideally pinned memory via a
    torch CPU tensor's numpy view): one synchronous C call does H2D, R-NW, device CRT and D2H;
    the returned words are marshalled to Python ints.  `out` (uint32 [count, KMAX + 3]) may be
    passed to reuse a (pinned) result buffer."""
    a = np.asarray(h_mats)
    if a.dtype != np.int32 or not a.flags.c_contiguous or a.ndim != 3:
        raise TypeError("expected a C-contiguous int32 array [count, n, n]")
    count, n = int(a.shape[0]), int(a.shape[1])
    limbs = KMAX + 2
    if out is None:
        out = np.empty((count, limbs + 1), dtype=np.uint32)
    _check(lib().sperm_permanent_host(a.ctypes.data if a.size else None, n, count, int(min_primes),
                                      out.ctypes.data if count else None, limbs, _stream(stream)))
    mag, sign = out[:, :limbs], out[:, limbs].view(np.int32)
    small = (~mag[:, 2:].any(axis=1)).tolist()
    lo = (mag[:, 0].astype(np.uint64) | (mag[:, 1].astype(np.uint64) << np.uint64(32))).tolist()
    buf = np.ascontiguousarray(mag).tobytes()
    w = 4 * limbs
    return [s_ * (v if sm else int.from_bytes(buf[r * w:(r + 1) * w], "little"))
            for r, (s_, v, sm) in enumerate(zip(sign.tolist(), lo, small))]


def sperm_rnw_terms(n: int, count: int) -> float:
    return float(lib().sperm_rnw_terms(int(n), int(count)))


def sperm_rnw_stats(reset: bool = False):
    """(terms, fma_units, alu_ops) of the sperm_permanent calls since the last reset."""
    t, f, a = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().sperm_rnw_stats(ctypes.byref(t), ctypes.byref(f), ctypes.byref(a), 1 if reset else 0))
    return t.value, f.value, a.value


def sperm_reduce_mod(acc, stream=None):
    import torch
    acc = _dev(acc, torch.int64)
    rows = int(acc.shape[0])
    out = torch.empty((rows, KMAX), dtype=torch.int32, device=acc.device)
    _check(lib().sperm_reduce_mod(_ptr(acc), rows, _ptr(out), _stream(stream)))
    return out


def sperm_fold_mod(acc, stream=None):
    """acc[r][q] %= p_q in place (uint64 accumulators stored as int64)."""
    import torch
    if not (isinstance(acc, torch.Tensor) and acc.is_cuda and acc.dtype == torch.int64 and acc.is_contiguous()):
        raise TypeError("expected a contiguous int64 CUDA tensor")
    _check(lib().sperm_fold_mod(_ptr(acc), int(acc.shape[0]), _stream(stream)))
    return acc


def residues_to_ints_device(res, k, stream=None) -> List[int]:
    """residues_to_ints with the CRT on the GPU (sperm_crt_device): one device-to-host copy of
    [count][limbs + 1] words (magnitude limbs, sign), then marshalling to Python ints."""
    import torch
    res = _dev(res, torch.int32)
    count, stride = int(res.shape[0]), int(res.shape[1])
    if count == 0:
        return []
    k = _dev(k, torch.int32)
    limbs = KMAX + 2
    out = torch.empty((count, limbs + 1), dtype=torch.int32, device=res.device)
    st = stream if stream is not None else torch.cuda.current_stream(res.device)
    _check(lib().sperm_crt_device(_ptr(res), count, stride, _ptr(k), 0, _ptr(out), limbs, st.cuda_stream))
    # read-back into pinned memory (torch's host caching allocator) on the launching stream
    hp = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    with torch.cuda.stream(st):
        hp.copy_(out, non_blocking=True)
    st.synchronize()
    h = hp.numpy().view(np.uint32)
    mag, sign = h[:, :limbs], h[:, limbs].view(np.int32)
    small = (~mag[:, 2:].any(axis=1)).tolist()
    lo = (mag[:, 0].astype(np.uint64) | (mag[:, 1].astype(np.uint64) << np.uint64(32))).tolist()
    sg = sign.tolist()
    buf = np.ascontiguousarray(mag).tobytes()
    w = 4 * limbs
    return [s_ * (v if sm else int.from_bytes(buf[r * w:(r + 1) * w], "little"))
            for r, (s_, v, sm) in enumerate(zip(sg, lo, small))]


def residues_to_ints(res, k) -> List[int]:
    """CRT every row of a host/device residue table (uint32 stored as int32)."""
    import torch
    if isinstance(res, torch.Tensor):
        res = res.cpu().numpy()
    if isinstance(k, torch.Tensor):
        k = k.cpu().numpy()
    res = np.ascontiguousarray(np.asarray(res).view(np.uint32))
    count = res.shape[0]
    if count == 0:
        return []
    ks = np.ascontiguousarray(np.broadcast_to(np.asarray(k), (count,)).astype(np.int32))
    limbs = KMAX + 2
    mag = np.zeros((count, limbs), dtype=np.uint32)
    sign = np.zeros(count, dtype=np.int32)
    _check(lib().sperm_crt_batch(res.ctypes.data, count, res.shape[1], ks.ctypes.data, 0, mag.ctypes.data,
                                 limbs, sign.ctypes.data))
    # little-endian uint32 limbs -> Python ints (marshalling): values below 2^64 in one vectorized
    # step, the rest row by row
    small = (~mag[:, 2:].any(axis=1)).tolist()
    lo = (mag[:, 0].astype(np.uint64) | (mag[:, 1].astype(np.uint64) << np.uint64(32))).tolist()
    sg = sign.tolist()
    buf = mag.tobytes()
    w = 4 * mag.shape[1]
    return [s_ * (v if sm else int.from_bytes(buf[r * w:(r + 1) * w], "little"))
            for r, (s_, v, sm) in enumerate(zip(sg, lo, small))]


# --------------------------------------------------------------------- expansion
def sperm_expand(mats, coef=None, job=None, stream=None, ordered: bool = True):
    """One BFS level of Algorithm PH Step 2.  Returns ((mats, coef, job) of the
    children of order n-1, (mats, coef, job) of the unsplit s >= 5 nodes).
    ordered=False: sperm_expand_unordered (children in an unspecified order)."""
    import torch
    mats = _dev(mats, torch.int32)
    count, n = int(mats.shape[0]), int(mats.shape[1])
    dev = mats.device
    coef = _dev(coef, torch.int64)
    job = _dev(job, torch.int32)
    oc, ec = ctypes.c_int64(0), ctypes.c_int64(0)
    L = lib()
    fn = L.sperm_expand if ordered else L.sperm_expand_unordered
    # children are at most 2 per node: allocate that once; s >= 5 (early) nodes are rare, so
    # their buffer is sized by a second call only when the first reports them
    cap = 2 * count
    out = (torch.empty((cap, n - 1, n - 1), dtype=torch.int32, device=dev),
           torch.empty((cap,), dtype=torch.int64, device=dev), torch.empty((cap,), dtype=torch.int32, device=dev))
    rc = fn(_ptr(mats), _ptr(coef), _ptr(job), n, count, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]),
                        cap, None, None, None, 0, ctypes.byref(oc), ctypes.byref(ec), _stream(stream))
    if rc not in (OK, ERR_CAPACITY):
        _check(rc)
    no, ne = oc.value, ec.value
    early = (torch.empty((ne, n, n), dtype=torch.int32, device=dev),
             torch.empty((ne,), dtype=torch.int64, device=dev), torch.empty((ne,), dtype=torch.int32, device=dev))
    if rc == ERR_CAPACITY:
        _check(fn(_ptr(mats), _ptr(coef), _ptr(job), n, count, _ptr(out[0]), _ptr(out[1]),
                              _ptr(out[2]), cap, _ptr(early[0]), _ptr(early[1]), _ptr(early[2]), ne,
                              ctypes.byref(oc), ctypes.byref(ec), _stream(stream)))
    return (out[0][:no], out[1][:no], out[2][:no]), early


def sperm_expand_subtree(mats, leaf_order: int, cap: int, coef=None, job=None, stream=None):
    """H_per's recursion below the job level, depth first (sperm_expand_subtree): every node of
    mats [count, n, n] (n <= 32) expanded to its leaves of order `leaf_order` in one call.
    Returns ((mats, coef, job) of the leaves [*, L, L], (mats, coef, job) of the s >= 5 nodes
    met on the way, padded to order n), or None if more than `cap` leaves were produced (the
    caller re-runs on fewer nodes)."""
    import torch
    mats = _dev(mats, torch.int32)
    count, n = int(mats.shape[0]), int(mats.shape[1])
    dev = mats.device
    coef = _dev(coef, torch.int64)
    job = _dev(job, torch.int32)
    L = int(leaf_order)
    oc, ec = ctypes.c_int64(0), ctypes.c_int64(0)
    out = (torch.empty((cap, L, L), dtype=torch.int32, device=dev),
           torch.empty((cap,), dtype=torch.int64, device=dev), torch.empty((cap,), dtype=torch.int32, device=dev))
    fn = lib().sperm_expand_subtree
    args = (_ptr(mats), _ptr(coef), _ptr(job), n, count, L, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]), cap)
    rc = fn(*args, None, None, None, 0, ctypes.byref(oc), ctypes.byref(ec), _stream(stream))
    if rc == ERR_CAPACITY and oc.value > cap:
        return None
    if rc not in (OK, ERR_CAPACITY):
        _check(rc)
    ne = ec.value
    early = (torch.empty((ne, n, n), dtype=torch.int32, device=dev),
             torch.empty((ne,), dtype=torch.int64, device=dev), torch.empty((ne,), dtype=torch.int32, device=dev))
    if rc == ERR_CAPACITY:  # only the early nodes did not fit: the counts are exact
        _check(fn(*args, _ptr(early[0]), _ptr(early[1]), _ptr(early[2]), ne, ctypes.byref(oc), ctypes.byref(ec),
                  _stream(stream)))
    no = oc.value
    return (out[0][:no], out[1][:no], out[2][:no]), early


def sperm_expand_subtree_stats(reset: bool = False):
    """(algorithmic bytes, roots) of the sperm_expand_subtree calls since the last reset."""
    b, nn = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().sperm_expand_subtree_stats(ctypes.byref(b), ctypes.byref(nn), 1 if reset else 0))
    return b.value, nn.value


def sperm_expand_stats(reset: bool = False):
    """(algorithmic bytes, parent nodes) of the sperm_expand calls since the last reset."""
    b, nn = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().sperm_expand_stats(ctypes.byref(b), ctypes.byref(nn), 1 if reset else 0))
    return b.value, nn.value


def sperm_nnz(mats, stream=None):
    """Nonzeros of each matrix of mats [count, n, n] (int64 CUDA tensor [count])."""
    import torch
    mats = _dev(mats, torch.int32)
    count, n = int(mats.shape[0]), int(mats.shape[1])
    out = torch.empty((count,), dtype=torch.int64, device=mats.device)
    _check(lib().sperm_nnz(_ptr(mats), n, count, _ptr(out), _stream(stream)))
    return out


# --------------------------------------------------------------------- estimator
def sperm_estimate(mats, trials: int = 0, seed: int = 1, ids=None, keep_trials: bool = False, stream=None):
    """KKLLL estimates (fp64) of the 0/1 patterns of mats [count, n, n]."""
    import torch
    mats = _dev(mats, torch.int32)
    count, n = int(mats.shape[0]), int(mats.shape[1])
    if trials <= 0:
        trials = n * n
    est = torch.empty((count,), dtype=torch.float64, device=mats.device)
    xs = torch.empty((count, trials), dtype=torch.float64, device=mats.device) if keep_trials else None
    ids = _dev(ids, torch.int32)
    _check(lib().sperm_estimate(_ptr(mats), n, count, _ptr(ids), int(trials), int(seed) & (2**64 - 1),
                                _ptr(est), _ptr(xs), _stream(stream)))
    return (est, xs) if keep_trials else est


def sperm_estimate_stats(reset: bool = False):
    """(jobs through the frontal KKLLL kernel, jobs it handed to the CTA kernel) since the last reset."""
    a, b = ctypes.c_double(0), ctypes.c_double(0)
    _check(lib().sperm_estimate_stats(ctypes.byref(a), ctypes.byref(b), 1 if reset else 0))
    return a.value, b.value


# --------------------------------------------------------------------- schedule
POLICY = {"estimate": 0, "natural": 1, "random": 2}


def sperm_schedule(weights, machines: int, policy: str = "estimate", seed: int = 0):
    """Host LPT / list scheduling.  Returns (machine[count], order[count], loads[machines])."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    count = w.shape[0]
    machine = np.zeros(count, dtype=np.int32)
    order = np.zeros(count, dtype=np.int32)
    loads = np.zeros(machines, dtype=np.float64)
    _check(lib().sperm_schedule(w.ctypes.data if count else None, count, int(machines), POLICY[policy],
                                int(seed) & (2**64 - 1), machine.ctypes.data if count else None,
                                order.ctypes.data if count else None, loads.ctypes.data))
    return machine, order, loads


def sperm_interpolate_mod(values, xs, k: int):
    """Coefficients (mod the first k primes) of the polynomial through (xs[j], values[j] mod p_q):
    values uint32 [npts, >= k]; returns uint32 [npts, KMAX] (row t = coefficient of x^t)."""
    v = np.ascontiguousarray(np.asarray(values).view(np.uint32) if np.asarray(values).dtype == np.int32
                             else np.asarray(values, dtype=np.uint32))
    x = np.ascontiguousarray(np.asarray(xs, dtype=np.int64))
    npts = x.shape[0]
    out = np.zeros((npts, KMAX), dtype=np.uint32)
    _check(lib().sperm_interpolate_mod(v.ctypes.data, v.shape[1], x.ctypes.data, npts, int(k), out.ctypes.data, KMAX))
    return out


def sperm_list_schedule(cost, order, machines: int):
    """Algorithm LS replayed with actual costs: (machine[count], loads[machines])."""
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
    o = np.ascontiguousarray(np.asarray(order, dtype=np.int32))
    count = c.shape[0]
    machine = np.zeros(count, dtype=np.int32)
    loads = np.zeros(machines, dtype=np.float64)
    _check(lib().sperm_list_schedule(c.ctypes.data if count else None, o.ctypes.data if count else None, count,
                                     int(machines), machine.ctypes.data if count else None, loads.ctypes.data))
    return machine, loads


def replay_efficiency(cost, order, machines: int) -> float:
    """Parallel efficiency sum(T) / (m * makespan) of LS in `order` with actual costs T
    (Tables 5-7's efficiency)."""
    _, loads = sperm_list_schedule(cost, order, machines)
    mk = loads.max()
    return float(np.sum(cost) / (machines * mk)) if mk > 0 else 1.0


# --------------------------------------------------------------------- box-wide queue
QUEUE_HANDLE_BYTES = 64


class DeviceQueue:
    """The box-wide dynamic queue (sperm_queue_*): a uint64 counter in rank 0's device memory,
    mapped by the other ranks through CUDA IPC; claim(chunk) -> first index of the claimed range."""

    def __init__(self, handle: Optional[bytes] = None):
        import torch
        self.ptr = ctypes.c_void_p(0)
        self.owner = handle is None
        if self.owner:
            buf = ctypes.create_string_buffer(QUEUE_HANDLE_BYTES)
            _check(lib().sperm_queue_create(ctypes.byref(self.ptr), buf))
            self.handle = buf.raw
        else:
            buf = ctypes.create_string_buffer(bytes(handle), QUEUE_HANDLE_BYTES)
            _check(lib().sperm_queue_open(buf, ctypes.byref(self.ptr)))
            self.handle = bytes(handle)
        self.scratch = torch.zeros(1, dtype=torch.int64, device="cuda")
        # claims run on their own stream: a claim does not wait for the caller's queued work (the
        # rank claims its next chunk while the GPU finishes the current one's last kernels)
        self.stream = torch.cuda.Stream()

    def claim(self, chunk: int, stream=None) -> int:
        start = ctypes.c_int64(0)
        _check(lib().sperm_queue_claim(self.ptr, int(chunk), _ptr(self.scratch), ctypes.byref(start),
                                       _stream(stream if stream is not None else self.stream)))
        return start.value

    def close(self):
        if self.ptr:
            _check(lib().sperm_queue_close(self.ptr, 1 if self.owner else 0))
            self.ptr = ctypes.c_void_p(0)


# --------------------------------------------------------------------- statistics
def sperm_kendall_tau(x, y, return_counts: bool = False):
    """Kendall tau with Eq. (10)'s tie correction (host C++).  With return_counts also
    (S, T, U, m(m-1)/2)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
    if x.shape != y.shape or x.ndim != 1:
        raise ValueError("x and y must be 1-D of equal length")
    tau = ctypes.c_double(0)
    counts = np.zeros(4, dtype=np.int64)
    _check(lib().sperm_kendall_tau(x.ctypes.data if len(x) else None, y.ctypes.data if len(y) else None, len(x),
                                   ctypes.byref(tau), counts.ctypes.data))
    return (tau.value, tuple(int(c) for c in counts)) if return_counts else tau.value


def tau_z(tau: float, m: int) -> float:
    """Normal-approximation z score of tau under independence: E = 0, var = 2(2m+5)/(9m(m-1))
    (PAPER.md:406-409)."""
    import math
    return tau / math.sqrt(2.0 * (2 * m + 5) / (9.0 * m * (m - 1)))


# --------------------------------------------------------------------- timing
def sperm_launch_count(reset: bool = False) -> int:
    return int(lib().sperm_launch_count(1 if reset else 0))


def sperm_timing_enable(on: bool = True):
    lib().sperm_timing_enable(1 if on else 0)


def sperm_timing_reset():
    lib().sperm_timing_reset()


def sperm_timing_get(name: str) -> Tuple[float, int]:
    ms, n = ctypes.c_double(0), ctypes.c_int64(0)
    _check(lib().sperm_timing_get(name.encode(), ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value
