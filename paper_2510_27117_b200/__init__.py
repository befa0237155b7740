"""paper_2510_27117_b200 — B200-native GFORS hot path (arXiv 2510.27117).

Thin ctypes binding of ``libgfors.so`` (C ABI in include/gfors.h).  Argument marshalling only:
every step of the method runs in the library's sm_100a kernels.  There is no CPU fallback —
if the library is missing this module raises on import.

    s = Solver(device=0)
    s.load(inst)                  # gfors_load     (numpy arrays -> host, torch CUDA tensors -> device)
    s.preprocess()                # gfors_preprocess
    info = s.run(max_iters=...)   # gfors_run
    z, x, meta = s.best_incumbent()
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgfors.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -m paper_2510_27117_b200.build` "
        "(nvcc, sm_100a).  There is no CPU fallback."
    )
_lib = C.CDLL(LIB_PATH)

P = C.c_void_p
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double

STATUS = {0: "OK", 2: "NO_INCUMBENT", 3: "E_INPUT", 4: "E_DIVERGED", 5: "E_CUDA", 6: "E_NCCL", 7: "E_STATE", 8: "E_OOM"}


class GforsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gfors {STATUS.get(code, code)}: {msg}")
        self.code = code


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class DeviceOpts(C.Structure):
    _fields_ = [("device", I32), ("stream", P), ("rank", I32), ("world", I32), ("nccl_id", P), ("loopback", I32),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", P)]


def torch_allocator(device: int, stream=None):
    """(alloc, free) callbacks for gfors_device_opts backed by torch's caching allocator (the
    library's device buffers then show up in torch.cuda.memory_allocated and are reused by torch after
    the solver closes).  stream: the cudaStream_t the solver runs on (None: torch's current stream)."""
    import torch

    def _alloc(nbytes, _ctx):
        try:
            st = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
            return torch.cuda.caching_allocator_alloc(int(nbytes), device, st)
        except Exception:  # noqa: BLE001  (out of memory -> NULL -> GFORS_E_OOM)
            return None

    def _free(ptr, _ctx):
        torch.cuda.caching_allocator_delete(ptr)

    return ALLOC_FN(_alloc), FREE_FN(_free)


class Problem(C.Structure):
    _fields_ = [("n", I64), ("m", I64), ("mem_space", I32), ("k_rowptr", P), ("k_col", P), ("k_val", P),
                ("r", P), ("sense", P), ("q_rowptr", P), ("q_col", P), ("q_val", P), ("c", P),
                ("c0", D), ("maximize", I32)]


class PrepOpts(C.Structure):
    _fields_ = [("tol", D), ("max_iter", I32), ("precision", I32)]


class Scaling(C.Structure):
    _fields_ = [("obj_scale", D), ("k_scale", D), ("zero_rows", I64)]


class Params(C.Structure):
    _fields_ = [("sigma", D), ("k_int", I32), ("k_r", I32), ("k_b", I64),
                ("rho_min", D), ("rho_max", D), ("growth_T", D), ("growth_p", D), ("rho_delta", D),
                ("tol_primal", D), ("tol_dual", D), ("tol_binary", D), ("stall_rel", D),
                ("stall_window", I32), ("max_iters", I64), ("time_limit_s", D), ("seed", U64),
                ("use_graph", I32), ("trace_cap", I32),
                ("sampler", I32), ("a3_ls", I32), ("a3_n", I64), ("a3_gamma", D),
                ("relax", I32), ("repair", I32), ("complete", I32), ("row_shard", I32)]


class RunInfo(C.Structure):
    _fields_ = [("iters", I64), ("rounds", I64), ("candidates", I64), ("halt_reason", I32),
                ("elapsed_s", D), ("n_trace", I64), ("launches", I64)]


class IncumbentInfo(C.Structure):
    _fields_ = [("found_iter", I64), ("found_round", I64), ("found_index", I64), ("found_time_s", D),
                ("has_incumbent", I32)]


EXPORTS = {
    "gfors_params_default": (None, [C.POINTER(Params)]),
    "gfors_prep_opts_default": (None, [C.POINTER(PrepOpts)]),
    "gfors_create": (I32, [C.POINTER(P), C.POINTER(DeviceOpts)]),
    "gfors_load": (I32, [P, C.POINTER(Problem)]),
    "gfors_preprocess": (I32, [P, C.POINTER(PrepOpts), C.POINTER(Scaling)]),
    "gfors_run": (I32, [P, C.POINTER(Params), C.POINTER(RunInfo)]),
    "gfors_best_incumbent": (I32, [P, P, P, C.POINTER(IncumbentInfo)]),
    "gfors_last_error": (C.c_char_p, [P]),
    "gfors_destroy": (None, [P]),
    "gfors_get_scaled": (I32, [P, P, P, P]),
    "gfors_sample": (I32, [P, P, U64, C.c_uint32, I64, I64, P]),
    "gfors_eval": (I32, [P, P, I64, P, P]),
    "gfors_set_state": (I32, [P, P, P, P]),
    "gfors_get_state": (I32, [P, P, P, P]),
    "gfors_step": (I32, [P, I64, D, D, D]),
    "gfors_indicators": (I32, [P, D, D, D, P]),
    "gfors_get_trace": (I32, [P, P, I64, P]),
    "gfors_profile_blocks": (I32, [P, C.POINTER(Params), I32, P, I32, P]),
    "gfors_kernel_class_name": (C.c_char_p, [I32]),
    "gfors_profile_active": (I32, [P, P, P, I32]),
    "gfors_launches_per_block": (I64, [P, C.POINTER(Params)]),
    "gfors_merge_records": (I32, [P, P, P, I32]),
    "gfors_tu_reformulate": (I32, [P, P, P, I64]),
    "gfors_dims": (I32, [P, P, P, P]),
    "gfors_sample_assign3d": (I32, [P, P, U64, C.c_uint32, I64, I64, I64, D, I64, P]),
    "gfors_set_relax": (I32, [P, I32]),
    "gfors_repair": (I32, [P, P, I64]),
    "gfors_cover_complete": (I32, [P, P, P, I64]),
    "gfors_nccl_unique_id": (I32, [P]),
    "gfors_graph_note": (C.c_char_p, [P]),
    "gfors_set_option": (I32, [P, C.c_char_p, I64]),
    "gfors_sample_eval_timed": (I32, [P, P, U64, I64, I32, P]),
    "gfors_release_memory": (I32, [I32]),
}
for _name, (_res, _args) in EXPORTS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def lib():
    return _lib


def default_params(**kw) -> Params:
    p = Params()
    _lib.gfors_params_default(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown parameter {k!r}")
        setattr(p, k, v)
    return p


def release_memory(device: int = 0):
    """gfors_release_memory: return the library pool's memory on `device` (no solver of it alive)."""
    rc = _lib.gfors_release_memory(int(device))
    if rc != 0:
        raise GforsError(rc, "gfors_release_memory: a solver of the device is alive, or a bad device")


def merge_records(z, index, valid):
    """Host-side cross-rank incumbent merge rule of the library (no GPU needed)."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    idx = np.ascontiguousarray(index, dtype=np.int64)
    v = np.ascontiguousarray(valid, dtype=np.int32)
    return int(_lib.gfors_merge_records(z.ctypes.data_as(P), idx.ctypes.data_as(P), v.ctypes.data_as(P), len(z)))


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor
        return P(a.data_ptr())
    return a.ctypes.data_as(P)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for Solver(..., nccl_id=...) (create on one rank, broadcast)."""
    buf = (C.c_char * 128)()
    rc = _lib.gfors_nccl_unique_id(C.cast(buf, P))
    if rc != 0:
        raise GforsError(rc, "ncclGetUniqueId failed / libnccl.so.2 not loadable")
    return bytes(buf)


class Solver:
    """One gfors context on one GPU.  rank/world shard the samples; nccl_id (bytes from
    nccl_unique_id(), identical on all ranks) enables the in-loop incumbent exchange."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 loopback: bool = False, options: dict | None = None, allocator=None):
        """allocator: None (the library's private pool), "torch" (torch's caching allocator) or an
        (alloc, free) pair of ALLOC_FN / FREE_FN callbacks."""
        self._nccl_buf = (C.c_char * 128).from_buffer_copy(nccl_id) if nccl_id else None
        if allocator == "torch":
            import torch
            if not stream:  # the solver's stream and the allocator's must agree (stream-ordered reuse)
                stream = torch.cuda.current_stream(device).cuda_stream
            allocator = torch_allocator(device, stream)
        self._alloc_cb = allocator  # the callbacks must outlive the context
        opts = DeviceOpts(device, P(stream) if stream else None, rank, world,
                          C.cast(self._nccl_buf, P) if nccl_id else None, int(bool(loopback)),
                          allocator[0] if allocator else ALLOC_FN(), allocator[1] if allocator else FREE_FN(), None)
        h = P()
        rc = _lib.gfors_create(C.byref(h), C.byref(opts))
        if rc != 0:
            raise GforsError(rc, "gfors_create failed")
        self.h = h
        self.n = self.m = 0
        for k, v in (options or {}).items():  # gfors_set_option (load-time choices apply to the next load)
            self.set_option(k, v)

    def close(self):
        if getattr(self, "h", None):
            _lib.gfors_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc, ok=(0,)):
        if rc not in ok:
            raise GforsError(rc, _lib.gfors_last_error(self.h).decode())
        return rc

    # ------------------------------------------------------------------ boundary calls
    def load(self, inst: dict):
        """gfors_load.  inst: dict of the user-form arrays (see gen/instances.py).  numpy arrays are
        passed as host memory; torch CUDA tensors as device memory (all arrays must agree)."""
        keep = []
        tensors = {k: v for k, v in inst.items() if hasattr(v, "is_cuda")}
        is_dev = any(v.is_cuda for v in tensors.values())
        if is_dev:
            host = [k for k in ("k_rowptr", "k_col", "k_val", "r", "sense", "q_rowptr", "q_col", "q_val", "c")
                    if inst.get(k) is not None and not (k in tensors and tensors[k].is_cuda)]
            if host:
                raise ValueError(f"load: mixed host and device inputs ({', '.join(host)} not CUDA tensors)")
            import torch
            torch.cuda.current_stream().synchronize()  # inputs written on a torch stream are complete

        _TORCH_DT = {np.int64: "int64", np.int32: "int32", np.float64: "float64", np.int8: "int8"}

        def arr(key, dt):
            v = inst.get(key)
            if v is None:
                return None
            if is_dev:
                import torch
                want = getattr(torch, _TORCH_DT[dt])
                if v.dtype != want or not v.is_contiguous():
                    v = v.to(dtype=want).contiguous()  # the C ABI element types (include/gfors.h)
                keep.append(v)
                return v
            a = np.ascontiguousarray(v, dtype=dt)
            keep.append(a)
            return a

        pr = Problem()
        pr.n, pr.m = int(inst["n"]), int(inst["m"])
        pr.mem_space = 1 if is_dev else 0
        pr.k_rowptr = _ptr(arr("k_rowptr", np.int64))
        pr.k_col = _ptr(arr("k_col", np.int32))
        pr.k_val = _ptr(arr("k_val", np.float64))
        pr.r = _ptr(arr("r", np.float64))
        pr.sense = _ptr(arr("sense", np.int8))
        pr.q_rowptr = _ptr(arr("q_rowptr", np.int64))
        pr.q_col = _ptr(arr("q_col", np.int32))
        pr.q_val = _ptr(arr("q_val", np.float64))
        pr.c = _ptr(arr("c", np.float64))
        pr.c0 = float(inst.get("c0", 0.0))
        pr.maximize = int(bool(inst.get("maximize", False)))
        self._chk(_lib.gfors_load(self.h, C.byref(pr)))
        self.n, self.m = pr.n, pr.m
        self.n_orig = pr.n
        return self

    def tu_reformulate(self, rows_J, cols_I):
        """gfors_tu_reformulate (PAPER §2.4.1): eliminate x_I through the equality rows J."""
        J = np.ascontiguousarray(rows_J, dtype=np.int64)
        I = np.ascontiguousarray(cols_I, dtype=np.int32)
        self._chk(_lib.gfors_tu_reformulate(self.h, _ptr(J), _ptr(I), len(J)))
        n, m, no = I64(), I64(), I64()
        self._chk(_lib.gfors_dims(self.h, C.byref(n), C.byref(m), C.byref(no)))
        self.n, self.m, self.n_orig = n.value, m.value, no.value
        return self

    def preprocess(self, tol=1e-7, max_iter=500, precision=64):
        o = PrepOpts(tol, max_iter, precision)
        sc = Scaling()
        self._chk(_lib.gfors_preprocess(self.h, C.byref(o), C.byref(sc)))
        return {"obj_scale": sc.obj_scale, "k_scale": sc.k_scale, "zero_rows": sc.zero_rows}

    def run(self, params: Params | None = None, **kw):
        p = params or default_params(**kw)
        info = RunInfo()
        rc = _lib.gfors_run(self.h, C.byref(p), C.byref(info))
        res = {f: getattr(info, f) for f, _ in RunInfo._fields_}
        if rc == 4:
            res["diverged"] = True
            return res
        self._chk(rc)
        res["diverged"] = False
        return res

    def best_incumbent(self, want_x=True):
        z = C.c_double()
        x = np.zeros(getattr(self, "n_orig", self.n), dtype=np.uint8) if want_x else None
        info = IncumbentInfo()
        self._chk(_lib.gfors_best_incumbent(self.h, C.byref(z), _ptr(x), C.byref(info)), ok=(0, 2))
        meta = {f: getattr(info, f) for f, _ in IncumbentInfo._fields_}
        return z.value, x, meta

    # ------------------------------------------------------------------ test / bench hooks
    def scaled(self):
        s = np.zeros(self.m); r = np.zeros(self.m); c = np.zeros(self.n)
        self._chk(_lib.gfors_get_scaled(self.h, _ptr(s), _ptr(r), _ptr(c)))
        return s, r, c

    def sample(self, p, seed, round_id, word_begin, n_words):
        p = np.ascontiguousarray(p, dtype=np.float64)
        bits = np.zeros((self.n, n_words), dtype=np.uint64)
        self._chk(_lib.gfors_sample(self.h, _ptr(p), seed, round_id, word_begin, n_words, _ptr(bits)))
        return bits

    def sample_assign3d(self, p, seed, round_id, word_begin, n_words, a3_n, gamma=4.0, L=None):
        p = np.ascontiguousarray(p, dtype=np.float64)
        bits = np.zeros((self.n, n_words), dtype=np.uint64)
        self._chk(_lib.gfors_sample_assign3d(self.h, _ptr(p), seed, round_id, word_begin, n_words, a3_n,
                                             float(gamma), -1 if L is None else int(L), _ptr(bits)))
        return bits

    def set_relax(self, relax):
        self._chk(_lib.gfors_set_relax(self.h, int(relax)))

    def repair(self, bits):
        bits = np.array(bits, dtype=np.uint64, copy=True)
        self._chk(_lib.gfors_repair(self.h, _ptr(bits), bits.shape[1]))
        return bits

    def cover_complete(self, p, bits):
        p = np.ascontiguousarray(p, dtype=np.float64)
        bits = np.array(bits, dtype=np.uint64, copy=True)
        self._chk(_lib.gfors_cover_complete(self.h, _ptr(p), _ptr(bits), bits.shape[1]))
        return bits

    def eval(self, bits):
        bits = np.ascontiguousarray(bits, dtype=np.uint64)
        nw = bits.shape[1]
        feas = np.zeros(64 * nw, dtype=np.uint8)
        z = np.zeros(64 * nw)
        self._chk(_lib.gfors_eval(self.h, _ptr(bits), nw, _ptr(feas), _ptr(z)))
        return feas, z

    def set_state(self, x, xbar, y):
        a = [np.ascontiguousarray(v, dtype=np.float64) for v in (x, xbar, y)]
        self._chk(_lib.gfors_set_state(self.h, _ptr(a[0]), _ptr(a[1]), _ptr(a[2])))

    def get_state(self):
        x = np.zeros(self.n); xb = np.zeros(self.n); y = np.zeros(self.m)
        self._chk(_lib.gfors_get_state(self.h, _ptr(x), _ptr(xb), _ptr(y)))
        return x, xb, y

    def step(self, iters, rho, tau1, tau2):
        self._chk(_lib.gfors_step(self.h, iters, rho, tau1, tau2))

    def indicators(self, rho, tau1, tau2):
        out = np.zeros(4)
        self._chk(_lib.gfors_indicators(self.h, rho, tau1, tau2, _ptr(out)))
        return {"primal_gap": out[0], "sx": out[1], "sy": out[2], "dual_gap": out[1] + out[2],
                "binary_gap": out[3]}

    def trace(self, max_rows=1 << 20):
        rows = np.zeros((max_rows, 8))
        nr = C.c_int64()
        self._chk(_lib.gfors_get_trace(self.h, _ptr(rows), max_rows, C.byref(nr)))
        return rows[: nr.value]

    def profile_blocks(self, blocks, params: Params | None = None, **kw):
        p = params or default_params(**kw)
        ms = np.zeros(16)
        nc = C.c_int32()
        self._chk(_lib.gfors_profile_blocks(self.h, C.byref(p), blocks, _ptr(ms), 16, C.byref(nc)))
        return {_lib.gfors_kernel_class_name(k).decode(): float(ms[k]) for k in range(nc.value)}

    def profile_active(self):
        """(total active ms, active launches) per kernel class of the last profile_blocks call."""
        ams = np.zeros(16); an = np.zeros(16)
        self._chk(_lib.gfors_profile_active(self.h, _ptr(ams), _ptr(an), 16))
        return {_lib.gfors_kernel_class_name(k).decode(): (float(ams[k]), int(an[k])) for k in range(16)
                if _lib.gfors_kernel_class_name(k).decode()}

    def sample_eval_timed(self, p, seed, n_words, rounds):
        """gfors_sample_eval_timed: device ms of `rounds` sampling + evaluation rounds at fixed p."""
        p = np.ascontiguousarray(p, dtype=np.float64)
        ms = D()
        self._chk(_lib.gfors_sample_eval_timed(self.h, _ptr(p), int(seed), int(n_words), int(rounds), C.byref(ms)))
        return ms.value

    def set_option(self, key: str, value: int):
        """gfors_set_option (test/benchmark options, include/gfors.h)."""
        self._chk(_lib.gfors_set_option(self.h, key.encode(), int(value)))
        return self

    def graph_note(self):
        return _lib.gfors_graph_note(self.h).decode()

    def launches_per_block(self, params: Params | None = None, **kw):
        p = params or default_params(**kw)
        return int(_lib.gfors_launches_per_block(self.h, C.byref(p)))


def solve(inst, precision=64, device=0, **params):
    """Convenience: load -> preprocess -> run -> best_incumbent."""
    s = Solver(device)
    s.load(inst)
    s.preprocess(precision=precision)
    info = s.run(**params)
    z, x, meta = s.best_incumbent()
    return z, x, info, meta
