"""ctypes view of the CPU fp64 oracle (oracle/adx_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package.  It restates the reference's algorithm (Route B);
each C function cites the reference file:line it follows.  Parity of the
oracle itself is pinned by the reference's goldens in
tests/test_oracle_golden.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "libadx_oracle.so")

OR_OK, OR_INVALID_ARGUMENT, OR_OUT_OF_RANGE, OR_DOMAIN, OR_RUNTIME, OR_LOGIC = range(6)
_EXC = {
    OR_INVALID_ARGUMENT: ValueError,
    OR_OUT_OF_RANGE: IndexError,
    OR_DOMAIN: ArithmeticError,
    OR_RUNTIME: RuntimeError,
    OR_LOGIC: AssertionError,
}


def build() -> str:
    """Compile the oracle (gcc) if missing or stale."""
    src = [os.path.join(_HERE, f) for f in ("adx_oracle.c", "adx_oracle.h", "Makefile")]
    if not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        i, d, u64, ll = C.c_int, C.c_double, C.c_uint64, C.c_longlong
        P = C.POINTER
        L.or_last_error.restype = C.c_char_p
        L.or_rng_uniform.restype = d
        L.or_rng_normal.restype = d
        L.or_rng_next_u64.restype = u64
        L.or_rng_below.restype = u64
        L.or_rng_below.argtypes = [C.c_void_p, u64]
        L.or_rng_seed.argtypes = [C.c_void_p, u64]
        L.or_mix_seed.restype = u64
        L.or_mix_seed.argtypes = [u64, u64]
        L.or_random_normals.argtypes = [u64, i, P(d)]
        L.or_build_schedule.argtypes = [i, d, d, i, P(d), P(d), P(d)]
        L.or_ddim_step.argtypes = [P(d), P(d), i, i, P(d), i, P(d)]
        L.or_forward_diffuse.argtypes = [P(d), P(d), i, i, P(d), i, P(d)]
        L.or_model_build_toy.argtypes = [i, P(i), i, u64, i, P(C.c_void_p)]
        L.or_model_shell.argtypes = [i, P(i), P(i), i, i, P(C.c_void_p)]
        L.or_model_free.argtypes = [C.c_void_p]
        L.or_model_num_stages.argtypes = [C.c_void_p]
        L.or_model_num_links.argtypes = [C.c_void_p]
        L.or_model_links.argtypes = [C.c_void_p, P(i)]
        L.or_model_stage_macs.restype = ll
        L.or_model_stage_macs.argtypes = [C.c_void_p, i]
        L.or_model_set_stage_macs.argtypes = [C.c_void_p, i, ll]
        L.or_model_tensor.restype = P(d)
        L.or_model_tensor.argtypes = [C.c_void_p, i, i, P(i), P(i)]
        L.or_sinusoid.argtypes = [i, i, P(d)]
        L.or_eval_full.argtypes = [C.c_void_p, P(d), i, P(d)]
        L.or_stage_forward.argtypes = [C.c_void_p, i, P(d), i, i, P(d)]
        L.or_embed.argtypes = [C.c_void_p, i, P(d)]
        L.or_partition_balanced.argtypes = [P(ll), i, i, i, P(i), P(ll)]
        L.or_plan_async_flat.argtypes = [i, i, i, i, i, P(i), i, P(i)]
        L.or_run_serial.argtypes = [C.c_void_p, P(i), i, P(i), P(d), i, P(d), P(d), P(d), P(i), P(i)]
        L.or_run_parallel.argtypes = [C.c_void_p, P(i), i, P(i), P(d), i, P(d), P(d), P(d), P(d)]
        L.or_sequential_denoise.argtypes = [C.c_void_p, P(d), i, P(d), P(d), P(d)]
        L.or_compare_trajectories.argtypes = [P(d), P(d), i, i, P(d), P(d), P(d)]
        _lib = L
    return _lib


def _chk(rc: int) -> None:
    if rc != OR_OK:
        raise _EXC.get(rc, RuntimeError)(lib().or_last_error().decode())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


# ---------------------------------------------------------------- RNG
class Rng:
    """rng.hpp:12-60 (mt19937_64 + explicit uniform / Box-Muller / below)."""

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(312 * 8 + 64)
        lib().or_rng_seed(self._buf, C.c_uint64(seed))

    def next_u64(self) -> int:
        return lib().or_rng_next_u64(self._buf)

    def uniform(self) -> float:
        return lib().or_rng_uniform(self._buf)

    def normal(self) -> float:
        return lib().or_rng_normal(self._buf)

    def below(self, n: int) -> int:
        return lib().or_rng_below(self._buf, C.c_uint64(n))


def mix_seed(a: int, b: int) -> int:
    return lib().or_mix_seed(a, b)


def random_normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().or_random_normals(C.c_uint64(seed), n, _dp(out))
    return out


# ---------------------------------------------------------------- schedule
@dataclass
class Schedule:
    T: int
    betas: np.ndarray
    alphas: np.ndarray
    alpha_bars: np.ndarray


def build_schedule(T: int, beta_start: float, beta_end: float, kind: str = "linear") -> Schedule:
    k = {"linear": 0, "scaled-linear": 1}[kind]
    b = np.empty(max(T, 1)); a = np.empty(max(T, 1)); ab = np.empty(max(T, 1) + 1)
    _chk(lib().or_build_schedule(T, beta_start, beta_end, k, _dp(b), _dp(a), _dp(ab)))
    return Schedule(T, b, a, ab)


def ddim_step(x: np.ndarray, eps: np.ndarray, t: int, alpha_bars: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64); eps = np.ascontiguousarray(eps, np.float64)
    ab = np.ascontiguousarray(alpha_bars, np.float64)
    out = np.empty_like(x)
    _chk(lib().or_ddim_step(_dp(x), _dp(eps), x.size, t, _dp(ab), ab.size - 1, _dp(out)))
    return out


def forward_diffuse(x0, noise, t, alpha_bars):
    x0 = np.ascontiguousarray(x0, np.float64); noise = np.ascontiguousarray(noise, np.float64)
    ab = np.ascontiguousarray(alpha_bars, np.float64)
    out = np.empty_like(x0)
    _chk(lib().or_forward_diffuse(_dp(x0), _dp(noise), x0.size, t, _dp(ab), ab.size - 1, _dp(out)))
    return out


def sinusoid(t: int, dim: int) -> np.ndarray:
    out = np.empty(dim)
    lib().or_sinusoid(t, dim, _dp(out))
    return out


# ---------------------------------------------------------------- model
PROJ, W1, B1, TIN, W2, B2 = range(6)


class Model:
    """LayeredDenoiser restated (denoiser.hpp:29-72); tensors are numpy views
    (Eigen column-major storage, so arrays come back Fortran-ordered)."""

    def __init__(self, handle, L: int, widths, E: int):
        self._h = C.c_void_p(handle)
        self.L, self.widths, self.E = L, list(widths), E
        self.d = widths[0]

    @classmethod
    def build_toy(cls, L, widths, skip_spec="unet-mirror", seed=0, E=8):
        w = np.ascontiguousarray(widths, np.int32)
        h = C.c_void_p()
        spec = {"none": 0, "unet-mirror": 1}[skip_spec]
        _chk(lib().or_model_build_toy(L, _ip(w), spec, C.c_uint64(seed), E, C.byref(h)))
        return cls(h.value, L, widths, E)

    @classmethod
    def shell(cls, L, widths, links, E=2):
        w = np.ascontiguousarray(widths, np.int32)
        lk = np.ascontiguousarray(np.array(links, np.int32).reshape(-1), np.int32)
        if lk.size == 0:
            lk = np.zeros(2, np.int32)
        h = C.c_void_p()
        _chk(lib().or_model_shell(L, _ip(w), _ip(lk), len(links), E, C.byref(h)))
        return cls(h.value, L, widths, E)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().or_model_free(self._h)
            self._h = C.c_void_p()

    @property
    def links(self):
        n = lib().or_model_num_links(self._h)
        buf = np.zeros(max(2 * n, 2), np.int32)
        lib().or_model_links(self._h, _ip(buf))
        return [(int(buf[2 * k]), int(buf[2 * k + 1])) for k in range(n)]

    def stage_macs(self, stage: int) -> int:
        return lib().or_model_stage_macs(self._h, stage)

    def set_stage_macs(self, stage: int, macs: int) -> None:
        lib().or_model_set_stage_macs(self._h, stage, macs)

    def costs(self):
        return [self.stage_macs(s) for s in range(1, self.L + 1)]

    def tensor(self, stage: int, which: int) -> np.ndarray:
        r, c = C.c_int(), C.c_int()
        p = lib().or_model_tensor(self._h, stage, which, C.byref(r), C.byref(c))
        n = r.value * c.value
        arr = np.ctypeslib.as_array(p, shape=(n,))
        return arr.reshape((r.value, c.value), order="F")

    def stage_forward(self, stage: int, u, t: int) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(self.widths[stage])
        _chk(lib().or_stage_forward(self._h, stage, _dp(u), u.size, t, _dp(out)))
        return out

    def embed(self, t: int) -> np.ndarray:
        out = np.empty(self.E)
        lib().or_embed(self._h, t, _dp(out))
        return out

    def eval_full(self, x, t: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.d)
        _chk(lib().or_eval_full(self._h, _dp(x), t, _dp(out)))
        return out


# ---------------------------------------------------------------- partition / plan
def partition_balanced(costs, N: int, strategy: str = "sequential-balanced"):
    """Returns (stage_segment[L] 1-based, seg_macs[N])."""
    c = np.ascontiguousarray(costs, np.int64)
    L = c.size
    ss = np.zeros(L, np.int32)
    sm = np.zeros(max(N, 1), np.int64)
    st = {"sequential-balanced": 0, "first-last-grouped": 1}[strategy]
    _chk(lib().or_partition_balanced(c.ctypes.data_as(C.POINTER(C.c_longlong)), L, N, st, _ip(ss),
                                     sm.ctypes.data_as(C.POINTER(C.c_longlong))))
    return ss, sm


def plan_async_flat(T: int, w: int, N: int, S: int, time_shift: bool = False) -> np.ndarray:
    cap = 64 + T * (8 + 7 * (N + 2))
    buf = np.zeros(cap, np.int32)
    n = C.c_int()
    _chk(lib().or_plan_async_flat(T, w, N, S, int(time_shift), _ip(buf), cap, C.byref(n)))
    return buf[: n.value].copy()


# ---------------------------------------------------------------- executor
def run_serial(model: Model, stage_segment, N, plan_flat, alpha_bars, x_T):
    T = len(alpha_bars) - 1
    ss = np.ascontiguousarray(stage_segment, np.int32)
    pf = np.ascontiguousarray(plan_flat, np.int32)
    ab = np.ascontiguousarray(alpha_bars, np.float64)
    x = np.ascontiguousarray(x_T, np.float64)
    lat = np.zeros((T + 1, model.d)); eps = np.zeros((T, model.d))
    n_rounds = int(pf[6])
    se = np.zeros(max(n_rounds, 1), np.int32)
    bc = C.c_int()
    _chk(lib().or_run_serial(model._h, _ip(ss), N, _ip(pf), _dp(ab), T, _dp(x), _dp(lat), _dp(eps),
                             _ip(se), C.byref(bc)))
    return lat, eps, se[:n_rounds].tolist(), bc.value


def run_parallel(model: Model, stage_segment, N, plan_flat, alpha_bars, x_T):
    T = len(alpha_bars) - 1
    ss = np.ascontiguousarray(stage_segment, np.int32)
    pf = np.ascontiguousarray(plan_flat, np.int32)
    ab = np.ascontiguousarray(alpha_bars, np.float64)
    x = np.ascontiguousarray(x_T, np.float64)
    lat = np.zeros((T + 1, model.d)); eps = np.zeros((T, model.d))
    wall = C.c_double()
    _chk(lib().or_run_parallel(model._h, _ip(ss), N, _ip(pf), _dp(ab), T, _dp(x), _dp(lat), _dp(eps),
                               C.byref(wall)))
    return lat, eps, wall.value


def sequential_denoise(model: Model, alpha_bars, x_T):
    T = len(alpha_bars) - 1
    ab = np.ascontiguousarray(alpha_bars, np.float64)
    x = np.ascontiguousarray(x_T, np.float64)
    lat = np.zeros((T + 1, model.d)); eps = np.zeros((T, model.d))
    _chk(lib().or_sequential_denoise(model._h, _dp(ab), T, _dp(x), _dp(lat), _dp(eps)))
    return lat, eps


def compare_trajectories(a: np.ndarray, b: np.ndarray):
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"compare_trajectories: length mismatch ({a.shape[0]} vs {b.shape[0]})")
    n, d = a.shape
    per = np.zeros(n); fm = C.c_double(); mx = C.c_double()
    lib().or_compare_trajectories(_dp(a), _dp(b), n, d, _dp(per), C.byref(fm), C.byref(mx))
    return per, fm.value, mx.value
