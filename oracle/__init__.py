"""ctypes wrapper of the fp64 CPU oracle (oracle/holo_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` and
``--impl reference`` legs) may import this package.  The product package
``paper_2004_04049_b200`` never imports it and shares no code with it.

Each wrapper names the C function (and through it the PAPER.md passage) it
calls.  Arrays are numpy; complex fields are ``complex128`` [n][n] row-major.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "holo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fcx-limited-range",
          "-fno-fast-math"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc if it is missing or older than the source."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_U8 = C.POINTER(C.c_uint8)
_U32 = C.POINTER(C.c_uint32)
_u64 = C.c_uint64
_i = C.c_int


def lib():
    global _lib
    with _lock:
        if _lib is None:
            h = C.CDLL(build())
            sig = {
                "or_splitmix64": (_u64, [_u64, _u64]),
                "or_angle_code": (C.c_uint32, [_u64, _u64]),
                "or_phase_f64_batch": (None, [_U32, _u64, _D]),
                "or_lut_build": (None, [_u64, _u64, _F]),
                "or_lut_index": (_u64, [_u64, _u64]),
                "or_apply_phase": (None, [_F, _i, _F, _u64, _u64, _D]),
                "or_apply_phase_prng": (None, [_F, _i, _u64, _u64, _D]),
                "or_apply_phase_prng_q": (None, [_F, _i, _u64, _u64, _i, _D]),
                "or_dft2_direct": (None, [_D, _D, _i, _i, _i]),
                "or_dft2_separable": (None, [_D, _D, _i, _i, _i]),
                "or_fft2": (_i, [_D, _i, _i]),
                "or_quantise_binary": (_i, [C.c_double]),
                "or_pack_bits": (None, [_U8, _i, _i, _U8]),
                "or_mse_m1": (C.c_double, [_D, _F, _i, _i, _i, _i, _i]),
                "or_mse_alpha": (C.c_double, [_D, _F, _i, _i, _i, _i, _i]),
                "or_ospr_subframe": (_i, [_F, _i, _F, _u64, _u64, _U8, _D, _D]),
                "or_replay_from_bits": (_i, [_U8, _i, _i, _D]),
                "or_ospr": (_i, [_F, _i, _i, _i, _F, _u64, _u64, _U8, _D, _D, _i, _i, _i, _i]),
                "or_gs_step": (_i, [_D, _F, _i, _i, _D, _D, _U8, _D, _D, _D, _i, _i, _i, _i]),
                "or_gs": (_i, [_F, _i, _i, _F, _u64, _u64, _i, _D, _U8, _D, _D, _D, _i, _i, _i, _i]),
                "or_is_prime": (_i, [_u64]),
                "or_next_prime_above": (_u64, [_u64]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _lut_arg(lut):
    if lut is None:
        return None, 0
    lut = _f32(lut).reshape(-1, 2)
    return lut, lut.shape[0]


# --- a0: phase pool -------------------------------------------------------------

def splitmix64(seed: int, k: int) -> int:
    return int(lib().or_splitmix64(seed, k))


def angle_code(seed: int, k: int) -> int:
    return int(lib().or_angle_code(seed, k))


def phase_f64(u) -> np.ndarray:
    """Recipe R-5 steps 1-4 in double: [m][2] (cos, sin) for 32-bit codes u."""
    u = np.ascontiguousarray(u, dtype=np.uint32).ravel()
    out = np.empty((u.size, 2), dtype=np.float64)
    lib().or_phase_f64_batch(_p(u, _U32), u.size, _p(out, _D))
    return out


def lut_build(seed: int, n_lut: int) -> np.ndarray:
    """The phase LUT, float32 [n_lut][2] = (cos, sin)."""
    out = np.empty((n_lut, 2), dtype=np.float32)
    lib().or_lut_build(seed, n_lut, _p(out, _F))
    return out


def lut_index(g: int, n_lut: int) -> int:
    return int(lib().or_lut_index(g, n_lut))


# --- a2: randomisation ----------------------------------------------------------

def apply_phase(T, lut, cursor: int) -> np.ndarray:
    """R = T * lut[(cursor + p) mod N_LUT]; lut None or empty = flat (R-6)."""
    T = _f32(T)
    n = T.shape[0]
    lut, L = _lut_arg(lut)
    R = np.empty((n, n), dtype=np.complex128)
    lib().or_apply_phase(_p(T, _F), n, _p(lut, _F), L, cursor, _p(R, _D))
    return R


def apply_phase_prng(T, seed: int, cursor: int) -> np.ndarray:
    T = _f32(T)
    n = T.shape[0]
    R = np.empty((n, n), dtype=np.complex128)
    lib().or_apply_phase_prng(_p(T, _F), n, seed, cursor, _p(R, _D))
    return R


def apply_phase_prng_q(T, seed: int, cursor: int, q: int) -> np.ndarray:
    """P:170 / R-25: the PRNG source with phases quantised to 2^q levels (a 2^q-entry
    sin/cos table): R = T * R5(u_g truncated to its top q bits)."""
    T = _f32(T)
    n = T.shape[0]
    R = np.empty((n, n), dtype=np.complex128)
    lib().or_apply_phase_prng_q(_p(T, _F), n, seed, cursor, q, _p(R, _D))
    return R


# --- A1-A3: DFT -------------------------------------------------------------------

def dft2_direct(f, inverse: bool = False) -> np.ndarray:
    f = _c128(f)
    ny, nx = f.shape
    out = np.empty_like(f)
    lib().or_dft2_direct(_p(f, _D), _p(out, _D), nx, ny, int(inverse))
    return out


def dft2_separable(f, inverse: bool = False) -> np.ndarray:
    f = _c128(f)
    ny, nx = f.shape
    out = np.empty_like(f)
    lib().or_dft2_separable(_p(f, _D), _p(out, _D), nx, ny, int(inverse))
    return out


def fft2(f, inverse: bool = False) -> np.ndarray:
    a = _c128(f).copy()
    if lib().or_fft2(_p(a, _D), a.shape[0], int(inverse)) != 0:
        raise ValueError("oracle fft2 needs a power-of-two square field")
    return a


# --- A5: quantisation -------------------------------------------------------------

def quantise_binary(re: float) -> int:
    return int(lib().or_quantise_binary(re))


def pack_bits(pm) -> np.ndarray:
    """pm: [ny][nx] of 1 (+1) / 0 (-1) -> [ny][ceil(nx/8)] MSB-first bytes."""
    pm = np.ascontiguousarray(pm, dtype=np.uint8)
    ny, nx = pm.shape
    out = np.empty((ny, (nx + 7) // 8), dtype=np.uint8)
    lib().or_pack_bits(_p(pm, _U8), nx, ny, _p(out, _U8))
    return out


# --- metrics ------------------------------------------------------------------------

def mse_m1(Iv, T, region) -> float:
    Iv = np.ascontiguousarray(Iv, dtype=np.float64)
    T = _f32(T)
    return float(lib().or_mse_m1(_p(Iv, _D), _p(T, _F), T.shape[0], *region))


def mse_alpha(Iv, T, region) -> float:
    Iv = np.ascontiguousarray(Iv, dtype=np.float64)
    T = _f32(T)
    return float(lib().or_mse_alpha(_p(Iv, _D), _p(T, _F), T.shape[0], *region))


# --- OSPR -----------------------------------------------------------------------------

def ospr_subframe(T, lut, cursor: int, want_h: bool = True, want_intensity: bool = True):
    """One sub-frame: returns (bits [n][n/8], Re H [n][n] or None, |F{H'}|^2 or None)."""
    T = _f32(T)
    n = T.shape[0]
    lut, L = _lut_arg(lut)
    bits = np.empty((n, n // 8), dtype=np.uint8)
    h = np.empty((n, n), dtype=np.float64) if want_h else None
    Iv = np.zeros((n, n), dtype=np.float64) if want_intensity else None
    rc = lib().or_ospr_subframe(_p(T, _F), n, _p(lut, _F), L, cursor, _p(bits, _U8), _p(h, _D), _p(Iv, _D))
    if rc:
        raise ValueError("bad size")
    return bits, h, Iv


def replay_from_bits(bits, n: int) -> np.ndarray:
    """Time-averaged replay intensity of packed sub-frames bits [n_sub][n][n/8]."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8).reshape(-1, n, n // 8)
    out = np.empty((n, n), dtype=np.float64)
    if lib().or_replay_from_bits(_p(bits, _U8), n, bits.shape[0], _p(out, _D)):
        raise ValueError("bad size")
    return out


def ospr(T, n_sub: int, lut, cursor0: int, region):
    """OSPR over frames T [F][n][n]: returns (bits [F][n_sub][n][n/8], intensity [F][n][n], mse [F])."""
    T = _f32(T)
    if T.ndim == 2:
        T = T[None]
    F, n, _ = T.shape
    lut, L = _lut_arg(lut)
    bits = np.empty((F, n_sub, n, n // 8), dtype=np.uint8)
    Iv = np.empty((F, n, n), dtype=np.float64)
    mse = np.empty(F, dtype=np.float64)
    rc = lib().or_ospr(_p(T, _F), n, F, n_sub, _p(lut, _F), L, cursor0, _p(bits, _U8), _p(Iv, _D),
                       _p(mse, _D), *region)
    if rc:
        raise ValueError("bad arguments")
    return bits, Iv, mse


# --- GS ---------------------------------------------------------------------------------

def gs_step(R_in, T, levels: int, region):
    """One GS iteration from R_{k-1}: returns dict(R, holo, levels, I, mse, E)."""
    R_in = _c128(R_in)
    T = _f32(T)
    n = T.shape[0]
    R = np.empty((n, n), dtype=np.complex128)
    h = np.empty((n, n), dtype=np.complex128)
    lev = np.zeros((n, n), dtype=np.uint8)
    Iv = np.empty((n, n), dtype=np.float64)
    mse = np.zeros(1)
    E = np.zeros(1)
    rc = lib().or_gs_step(_p(R_in, _D), _p(T, _F), n, levels, _p(R, _D), _p(h, _D), _p(lev, _U8),
                          _p(Iv, _D), _p(mse, _D), _p(E, _D), *region)
    if rc:
        raise ValueError("bad size")
    return {"R": R, "holo": h, "levels": lev, "I": Iv, "mse": float(mse[0]), "E": float(E[0])}


def gs(T, iters: int, lut, cursor: int, levels: int, region):
    """Full GS for one frame: returns dict(holo, levels, I, mse [iters], E [iters])."""
    T = _f32(T)
    n = T.shape[0]
    lut, L = _lut_arg(lut)
    h = np.empty((n, n), dtype=np.complex128)
    lev = np.zeros((n, n), dtype=np.uint8)
    Iv = np.empty((n, n), dtype=np.float64)
    mse = np.empty(iters)
    E = np.empty(iters)
    rc = lib().or_gs(_p(T, _F), n, iters, _p(lut, _F), L, cursor, levels, _p(h, _D), _p(lev, _U8),
                     _p(Iv, _D), _p(mse, _D), _p(E, _D), *region)
    if rc:
        raise ValueError("bad arguments")
    return {"holo": h, "levels": lev, "I": Iv, "mse": mse, "E": E}


# --- host utilities ------------------------------------------

def is_prime(m: int) -> bool:
    return bool(lib().or_is_prime(m))


def next_prime_above(m: int) -> int:
    return int(lib().or_next_prime_above(m))


def hard_limits(nx: int, ny: int, n_sf: int):
    """§5.1 / conclusion limits: (N_SF, Nx*Ny*N_SF, max(Nx, Ny))."""
    return (n_sf, nx * ny * n_sf, max(nx, ny))
