"""ctypes binding for the CPU oracle (oracle/gfors_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs may import this module.  It never touches the CUDA library and the CUDA library never
touches it.  Arithmetic lives in the C file; this file only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gfors_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no FMA contraction so expressions round as written)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "gfors_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-D_POSIX_C_SOURCE=200809L", "-ffp-contract=off", "-fno-fast-math",
             "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        )
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


P = C.c_void_p
I64 = C.c_int64
D = C.c_double


class OrcParams(C.Structure):
    _fields_ = [("sigma", D), ("k_int", C.c_int32), ("k_r", C.c_int32), ("k_b", I64),
                ("rho_min", D), ("rho_max", D), ("growth_T", D), ("growth_p", D), ("rho_delta", D),
                ("tol_primal", D), ("tol_dual", D), ("tol_binary", D), ("stall_rel", D),
                ("stall_window", C.c_int32), ("max_iters", I64), ("time_limit_s", D), ("seed", C.c_uint64),
                ("sampler", C.c_int32), ("a3_ls", C.c_int32), ("a3_n", I64), ("a3_gamma", D),
                ("relax", C.c_int32), ("repair", C.c_int32), ("complete", C.c_int32)]


class OrcRunInfo(C.Structure):
    _fields_ = [("iters", I64), ("rounds", I64), ("candidates", I64), ("halt_reason", C.c_int),
                ("found_iter", I64), ("found_round", I64), ("found_index", I64), ("has_incumbent", C.c_int),
                ("z_best", D)]


class OrcHaltState(C.Structure):
    _fields_ = [("tol", D * 3), ("stall_rel", D), ("window", C.c_int), ("count", C.c_int),
                ("hist", (D * 1024) * 3), ("since_improve", I64)]


def _declare(L):
    L.orc_philox4x32_10.argtypes = [P, P, P]
    L.orc_create.argtypes = [C.POINTER(P), I64, I64, P, P, P, P, P, P, P, P, P, D, C.c_int]
    L.orc_create.restype = C.c_int
    L.orc_destroy.argtypes = [P]
    L.orc_last_error.restype = C.c_char_p
    L.orc_info.argtypes = [P, P, P, P]
    L.orc_row_perm.argtypes = [P, P]
    L.orc_spectral_norm.argtypes = [I64, I64, P, P, P, D, C.c_int]
    L.orc_spectral_norm.restype = D
    L.orc_preprocess.argtypes = [P, D, C.c_int, P, P, P]
    L.orc_scaled_dense.argtypes = [P, P, P, P, P]
    L.orc_row_scales.argtypes = [P, P]
    L.orc_rho_schedule.argtypes = [D, D, D, D, D, I64, P]
    L.orc_state_init.argtypes = [P]
    L.orc_set_state.argtypes = [P, P, P, P]
    L.orc_get_state.argtypes = [P, P, P, P]
    L.orc_step.argtypes = [P, D, D, D]
    L.orc_indicators.argtypes = [P, D, D, D, P]
    L.orc_sample.argtypes = [P, I64, C.c_uint64, C.c_uint32, I64, I64, P]
    L.orc_sample_subset.argtypes = [P, P, I64, C.c_uint64, C.c_uint32, I64, I64, P]
    L.orc_sample_assign3d.argtypes = [P, I64, P, C.c_uint64, C.c_uint32, I64, I64, D, I64, P]
    L.orc_canonical_c.argtypes = [P, P]
    L.orc_set_relax.argtypes = [P, C.c_int]
    L.orc_repair.argtypes = [P, P, I64]
    L.orc_cover_complete.argtypes = [P, P, P, I64]
    L.orc_eval.argtypes = [P, P, I64, P, P]
    L.orc_eval_point.argtypes = [P, P, P, P]
    L.orc_halt_init.argtypes = [C.POINTER(OrcHaltState), D, D, D, D, C.c_int]
    L.orc_halt_push.argtypes = [C.POINTER(OrcHaltState), D, D, D, C.c_int]
    L.orc_halt_push.restype = C.c_int
    L.orc_params_default.argtypes = [C.POINTER(OrcParams)]
    L.orc_run.argtypes = [P, C.POINTER(OrcParams), C.POINTER(OrcRunInfo), P, I64, P]
    L.orc_best.argtypes = [P, P, P]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def spectral_norm(rowptr, col, val, rows, cols, tol=1e-7, max_iter=500):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    return lib().orc_spectral_norm(rows, cols, _ptr(rowptr), _ptr(col), _ptr(val), tol, max_iter)


def rho_schedule(rho_min, rho_max, T, p, delta, count):
    out = np.zeros(count, dtype=np.float64)
    lib().orc_rho_schedule(rho_min, rho_max, T, p, delta, count, _ptr(out))
    return out


def sample(p, seed, round_id, word_begin, n_words):
    p = np.ascontiguousarray(p, dtype=np.float64)
    bits = np.zeros((p.shape[0], n_words), dtype=np.uint64)
    lib().orc_sample(_ptr(p), p.shape[0], seed, round_id, word_begin, n_words, _ptr(bits))
    return bits


def sample_assign3d(p, a3n, cost, seed, round_id, word_begin, n_words, gamma=4.0, L=None):
    """Alg. 4 customised sampler (3D assignment).  cost: canonical (minimisation) c."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    assert p.shape[0] == a3n ** 3 == cost.shape[0]
    bits = np.zeros((p.shape[0], n_words), dtype=np.uint64)
    lib().orc_sample_assign3d(_ptr(p), a3n, _ptr(cost), seed, round_id, word_begin, n_words, float(gamma),
                              2 * a3n if L is None else int(L), _ptr(bits))
    return bits


def sample_subset(p_sub, idx, seed, round_id, word_begin, n_words):
    p_sub = np.ascontiguousarray(p_sub, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    bits = np.zeros((idx.shape[0], n_words), dtype=np.uint64)
    lib().orc_sample_subset(_ptr(p_sub), _ptr(idx), idx.shape[0], seed, round_id, word_begin, n_words, _ptr(bits))
    return bits


def params(**kw) -> OrcParams:
    p = OrcParams()
    lib().orc_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class HaltState:
    def __init__(self, tol_p=1e-6, tol_d=1e-6, tol_b=1e-6, stall_rel=1e-8, window=50):
        self.s = OrcHaltState()
        lib().orc_halt_init(C.byref(self.s), tol_p, tol_d, tol_b, stall_rel, window)

    def push(self, pg, dg, bg, improved):
        return bool(lib().orc_halt_push(C.byref(self.s), pg, dg, bg, int(bool(improved))))


class Oracle:
    """One canonicalised problem (user form in, see gfors_oracle.h)."""

    def __init__(self, inst: dict):
        L = lib()
        self._keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a

        n, m = int(inst["n"]), int(inst["m"])
        self.n, self.m = n, m
        h = P()
        rc = L.orc_create(C.byref(h), n, m,
                          _ptr(arr(inst.get("k_rowptr"), np.int64)), _ptr(arr(inst.get("k_col"), np.int32)),
                          _ptr(arr(inst.get("k_val"), np.float64)), _ptr(arr(inst.get("r"), np.float64)),
                          _ptr(arr(inst.get("sense"), np.int8)),
                          _ptr(arr(inst.get("q_rowptr"), np.int64)), _ptr(arr(inst.get("q_col"), np.int32)),
                          _ptr(arr(inst.get("q_val"), np.float64)), _ptr(arr(inst["c"], np.float64)),
                          float(inst.get("c0", 0.0)), int(bool(inst.get("maximize", False))))
        if rc != 0:
            raise ValueError(f"oracle load failed ({rc}): {L.orc_last_error().decode()}")
        self.h = h
        m1, m2, integ = I64(), I64(), C.c_int()
        L.orc_info(h, C.byref(m1), C.byref(m2), C.byref(integ))
        self.m1, self.m2, self.integral = m1.value, m2.value, bool(integ.value)
        self._keep = []

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_destroy(self.h)
            self.h = None

    def row_perm(self):
        out = np.zeros(self.m, dtype=np.int64)
        lib().orc_row_perm(self.h, _ptr(out))
        return out

    def preprocess(self, tol=1e-7, max_iter=500):
        a, b, z = D(), D(), I64()
        lib().orc_preprocess(self.h, tol, max_iter, C.byref(a), C.byref(b), C.byref(z))
        return {"obj_scale": a.value, "k_scale": b.value, "zero_rows": z.value}

    def scaled_dense(self):
        K = np.zeros((self.m, self.n)); r = np.zeros(self.m)
        Q = np.zeros((self.n, self.n)); c = np.zeros(self.n)
        self._chk(lib().orc_scaled_dense(self.h, _ptr(K), _ptr(r), _ptr(Q), _ptr(c)))
        return K, r, Q, c

    def row_scales(self):
        s = np.zeros(self.m)
        self._chk(lib().orc_row_scales(self.h, _ptr(s)))
        return s

    def state_init(self):
        self._chk(lib().orc_state_init(self.h))

    def set_state(self, x, xbar, y):
        x = np.ascontiguousarray(x, np.float64); xb = np.ascontiguousarray(xbar, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        self._chk(lib().orc_set_state(self.h, _ptr(x), _ptr(xb), _ptr(y)))

    def get_state(self):
        x = np.zeros(self.n); xb = np.zeros(self.n); y = np.zeros(self.m)
        self._chk(lib().orc_get_state(self.h, _ptr(x), _ptr(xb), _ptr(y)))
        return x, xb, y

    def step(self, rho, tau1, tau2):
        self._chk(lib().orc_step(self.h, rho, tau1, tau2))

    def indicators(self, rho, tau1, tau2):
        out = np.zeros(4)
        self._chk(lib().orc_indicators(self.h, rho, tau1, tau2, _ptr(out)))
        return {"primal_gap": out[0], "sx": out[1], "sy": out[2], "dual_gap": out[1] + out[2],
                "binary_gap": out[3]}

    def eval(self, bits):
        bits = np.ascontiguousarray(bits, dtype=np.uint64)
        nw = bits.shape[1]
        feas = np.zeros(64 * nw, dtype=np.uint8); z = np.zeros(64 * nw)
        self._chk(lib().orc_eval(self.h, _ptr(bits), nw, _ptr(feas), _ptr(z)))
        return feas, z

    def set_relax(self, relax):
        self._chk(lib().orc_set_relax(self.h, int(relax)))

    def repair(self, bits):
        bits = np.array(bits, dtype=np.uint64, copy=True)
        self._chk(lib().orc_repair(self.h, _ptr(bits), bits.shape[1]))
        return bits

    def cover_complete(self, p, bits):
        p = np.ascontiguousarray(p, dtype=np.float64)
        bits = np.array(bits, dtype=np.uint64, copy=True)
        self._chk(lib().orc_cover_complete(self.h, _ptr(p), _ptr(bits), bits.shape[1]))
        return bits

    def canonical_c(self):
        c = np.zeros(self.n)
        lib().orc_canonical_c(self.h, _ptr(c))
        return c

    def eval_point(self, x):
        x = np.ascontiguousarray(x, dtype=np.uint8)
        f, z = C.c_int(), D()
        self._chk(lib().orc_eval_point(self.h, _ptr(x), C.byref(f), C.byref(z)))
        return bool(f.value), z.value

    def run(self, prm: OrcParams | None = None, trace_max=0, **kw):
        prm = prm or params(**kw)
        info = OrcRunInfo()
        tr = np.zeros((max(trace_max, 1), 8))
        nt = I64()
        rc = lib().orc_run(self.h, C.byref(prm), C.byref(info), _ptr(tr), trace_max, C.byref(nt))
        if rc not in (0, -4):
            self._chk(rc)
        res = {f: getattr(info, f) for f, _ in OrcRunInfo._fields_}
        res["diverged"] = rc == -4
        res["trace"] = tr[: min(nt.value, trace_max)]
        return res

    def best(self):
        z = D(); x = np.zeros(self.n, dtype=np.uint8)
        lib().orc_best(self.h, C.byref(z), _ptr(x))
        return z.value, x

    @staticmethod
    def _chk(rc):
        if rc != 0:
            raise RuntimeError(f"oracle error {rc}: {lib().orc_last_error().decode()}")
