"""TEST INFRASTRUCTURE ONLY -- ctypes loader for the CPU oracle (oracle.c).

The oracle is the plain single-threaded fp64 CPU implementation of the SALE
per-cycle update as SURVEY.md §8(c) writes it down (arXiv 2209.01983 names the
steps, P:133/P:158/P:181/P:264, but prints no discrete equations).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(``paper_2209_01983_b200``) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
LIB_PATH = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared", "-Wall"]

OK, EINVAL, ENOMEM, ETANGLED, EDTCOLLAPSE, ENEGMASS, EPOISONED = 0, 1, 2, 5, 6, 7, 8

FIELDS = {"X": 0, "Y": 1, "Z": 2, "UX": 3, "UY": 4, "UZ": 5, "NODE_MASS": 6,
          "MASS": 7, "E": 8, "RHO": 9, "VOL": 10, "P": 11, "Q": 12, "CS": 13}
MAX_MAT = 4
for _m in range(MAX_MAT):  # material fields (nmat >= 1): volume fraction, mass, specific energy
    FIELDS[f"MAT_F{_m}"], FIELDS[f"MAT_M{_m}"], FIELDS[f"MAT_E{_m}"] = 16 + _m, 20 + _m, 24 + _m
NODE_FIELDS = ("X", "Y", "Z", "UX", "UY", "UZ", "NODE_MASS")


class OracleParams(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("nz", C.c_int32), ("lx", C.c_double), ("ly", C.c_double),
                ("lz", C.c_double), ("gamma", C.c_double), ("q_lin", C.c_double),
                ("q_quad", C.c_double), ("cfl", C.c_double), ("dt_growth", C.c_double),
                ("t_end", C.c_double), ("rezone", C.c_int32), ("reflect_mask", C.c_uint32),
                ("rho0", C.c_double), ("e_background", C.c_double),
                ("e_deposit", C.c_double), ("nmat", C.c_int32), ("pad0", C.c_int32),
                ("mat_gamma", C.c_double * 4), ("hg", C.c_double)]


_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -ffp-contract=off (no FMA contraction)."""
    stale = (not os.path.exists(LIB_PATH)
             or os.path.getmtime(LIB_PATH) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def use_openmp() -> str:
    """Switch this process to the -fopenmp build of the same source (liboracle_omp.so):
    the whole-mesh loops run on OMP_NUM_THREADS threads with bit-identical results
    (oracle.c header).  For the full-size golden digests only; call before lib()."""
    global LIB_PATH
    path = os.path.join(_HERE, "liboracle_omp.so")
    if not os.path.exists(path) or os.path.getmtime(path) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)):
        tmp = path + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, path)
    LIB_PATH = path
    return path


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.endswith("liboracle_omp.so"):
                build()
            L = C.CDLL(LIB_PATH)
            P = C.POINTER
            d, i32, i64, u64 = C.c_double, C.c_int32, C.c_int64, C.c_uint64
            vp = C.c_void_p
            L.oracle_create.argtypes = [P(OracleParams), P(vp)]
            L.oracle_create.restype = i32
            L.oracle_step.argtypes = [vp, i32, P(i32)]
            L.oracle_step.restype = i32
            L.oracle_get_field.argtypes = [vp, i32, P(d), u64]
            L.oracle_get_field.restype = i32
            L.oracle_set_field.argtypes = [vp, i32, P(d), u64]
            L.oracle_set_field.restype = i32
            L.oracle_get_clock.argtypes = [vp, P(d), P(d), P(i64), P(i32)]
            L.oracle_get_clock.restype = i32
            L.oracle_set_clock.argtypes = [vp, d, d, i64]
            L.oracle_set_clock.restype = i32
            L.oracle_last_error.argtypes = [vp]
            L.oracle_last_error.restype = C.c_char_p
            L.oracle_last_error_cell.argtypes = [vp]
            L.oracle_last_error_cell.restype = i64
            L.oracle_next_dt.argtypes = [vp, P(d)]
            L.oracle_next_dt.restype = i32
            L.oracle_steinberg_point.argtypes = [P(OracleSteinberg), d, d, d, d, P(d), P(d)]
            L.oracle_steinberg_point.restype = None
            L.oracle_steinberg.argtypes = [vp, P(OracleSteinberg), vp, P(d), P(d), u64]
            L.oracle_steinberg.restype = i32
            L.oracle_destroy.argtypes = [vp]
            L.oracle_destroy.restype = None
            L.oracle_face.argtypes = [P(d), P(d), P(d), P(d)]
            L.oracle_face.restype = None
            L.oracle_hex_volume.argtypes = [P(d)]
            L.oracle_hex_volume.restype = d
            L.oracle_eos.argtypes = [d, d, d, P(d), P(d), P(d)]
            L.oracle_eos.restype = None
            L.oracle_mix_eos.argtypes = [i32, P(d), P(d), P(d), P(d), d, d, P(d), P(d), P(d)]
            L.oracle_mix_eos.restype = None
            L.oracle_q_of_du.argtypes = [d, d, d, d, d]
            L.oracle_q_of_du.restype = d
            L.oracle_dt_cell.argtypes = [d, d, d, d, d, d, d]
            L.oracle_dt_cell.restype = d
            L.oracle_swept_volume.argtypes = [P(d), P(d)]
            L.oracle_swept_volume.restype = d
            L.oracle_cell_energy.argtypes = [P(d), P(d), P(d), d, d, d, d, d]
            L.oracle_cell_energy.restype = d
            L.oracle_hg_modes.argtypes = [P(d), P(d)]
            L.oracle_hg_modes.restype = None
            L.oracle_hg_corner.argtypes = [P(d), d, i32, P(d)]
            L.oracle_hg_corner.restype = None
            L.oracle_hg_nu.argtypes = [d, d, d, d, d]
            L.oracle_hg_nu.restype = d
            _lib = L
    return _lib


class OracleSteinberg(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("G0", "GP", "GT", "Y0", "Ymax", "beta", "n", "cv", "rho0", "T0")]


def steinberg_params(d: dict) -> OracleSteinberg:
    return OracleSteinberg(*[float(d[n]) for n, _ in OracleSteinberg._fields_])


def steinberg_point(params: dict, p, rho, e, eps_p=0.0):
    sh, y = C.c_double(), C.c_double()
    lib().oracle_steinberg_point(C.byref(steinberg_params(params)), p, rho, e, eps_p, C.byref(sh), C.byref(y))
    return sh.value, y.value


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_params(cfg: dict) -> OracleParams:
    p = OracleParams()
    p.abi_version = 3
    for name, _ in OracleParams._fields_:
        if name in ("abi_version", "pad0", "nmat", "mat_gamma", "hg"):
            continue
        setattr(p, name, cfg[name])
    p.hg = float(cfg.get("hg", 0.0))
    gam = list(cfg.get("mat_gamma", ()))[:4]  # nmat > 4 is rejected by oracle_create
    p.nmat = int(cfg.get("nmat", 0))
    p.mat_gamma = (C.c_double * 4)(*(gam + [0.0] * (4 - len(gam))))
    return p


class Oracle:
    """One oracle context (single rank, host memory)."""

    def __init__(self, cfg: dict):
        self.cfg = dict(cfg)
        self._L = lib()
        self._p = make_params(cfg)
        h = C.c_void_p()
        rc = self._L.oracle_create(C.byref(self._p), C.byref(h))
        if rc != OK:
            raise ValueError(f"oracle_create failed rc={rc}")
        self._h = h
        nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
        self.node_shape = (nz + 1, ny + 1, nx + 1)
        self.cell_shape = (nz, ny, nx)

    def close(self):
        if getattr(self, "_h", None):
            self._L.oracle_destroy(self._h)
            self._h = None

    __del__ = close

    def step(self, n: int):
        done = C.c_int32(0)
        rc = self._L.oracle_step(self._h, int(n), C.byref(done))
        return rc, done.value

    def get(self, field: str) -> np.ndarray:
        shape = self.node_shape if field in NODE_FIELDS else self.cell_shape
        out = np.empty(shape, dtype=np.float64)
        rc = self._L.oracle_get_field(self._h, FIELDS[field], _dp(out), out.size)
        if rc != OK:
            raise ValueError(f"oracle_get_field({field}) rc={rc}")
        return out

    def set(self, field: str, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, dtype=np.float64)
        rc = self._L.oracle_set_field(self._h, FIELDS[field], _dp(a), a.size)
        if rc != OK:
            raise ValueError(f"oracle_set_field({field}) rc={rc}")

    def clock(self):
        t, dt, cyc, fin = C.c_double(), C.c_double(), C.c_int64(), C.c_int32()
        self._L.oracle_get_clock(self._h, C.byref(t), C.byref(dt), C.byref(cyc), C.byref(fin))
        return {"t": t.value, "dt_last": dt.value, "cycle": cyc.value, "finished": fin.value}

    def set_clock(self, t: float, dt_last: float, cycle: int) -> None:
        rc = self._L.oracle_set_clock(self._h, t, dt_last, cycle)
        if rc != OK:
            raise ValueError(f"oracle_set_clock rc={rc}")

    def next_dt(self):
        dt = C.c_double()
        rc = self._L.oracle_next_dt(self._h, C.byref(dt))
        return rc, dt.value

    def steinberg(self, params, eps_p=None):
        """Shear modulus and yield stress of every cell (Fig. 6b; oracle.h).  params:
        one dict, or with a material axis a list of nmat dicts (outputs then gain a
        leading material axis)."""
        plist = list(params) if isinstance(params, (list, tuple)) else [params]
        if len(plist) != max(int(self.cfg.get("nmat", 0)), 1):
            raise ValueError("oracle_steinberg needs one parameter set per material")
        shape = ((len(plist),) + self.cell_shape) if isinstance(params, (list, tuple)) else self.cell_shape
        arr = (OracleSteinberg * len(plist))(*[steinberg_params(d) for d in plist])
        sh = np.empty(shape)
        y = np.empty(shape)
        e = None if eps_p is None else np.ascontiguousarray(eps_p, dtype=np.float64)
        rc = self._L.oracle_steinberg(self._h, C.cast(arr, C.POINTER(OracleSteinberg)),
                                      None if e is None else e.ctypes.data, _dp(sh), _dp(y), sh.size // len(plist))
        if rc != OK:
            raise ValueError(f"oracle_steinberg rc={rc}")
        return sh, y

    def last_error(self) -> str:
        return self._L.oracle_last_error(self._h).decode()

    def last_error_cell(self) -> int:
        return self._L.oracle_last_error_cell(self._h)


# ---- unit entry points ------------------------------------------------------
def face(P):
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(4, 3)
    A, Xb, s = np.zeros(3), np.zeros(3), C.c_double()
    lib().oracle_face(_dp(P), _dp(A), _dp(Xb), C.byref(s))
    return A, Xb, s.value


def hex_volume(N):
    N = np.ascontiguousarray(N, dtype=np.float64).reshape(8, 3)
    return lib().oracle_hex_volume(_dp(N))


def eos(gamma, rho, e):
    p, pf, cs = C.c_double(), C.c_double(), C.c_double()
    lib().oracle_eos(gamma, rho, e, C.byref(p), C.byref(pf), C.byref(cs))
    return p.value, pf.value, cs.value


def mix_eos(gammas, f, mm, e, V, rho):
    """MM1 mixed-cell closure: (p, P, cs) of one cell."""
    n = len(gammas)
    arr = [np.ascontiguousarray(a, dtype=np.float64) for a in (gammas, f, mm, e)]
    p, P, cs = C.c_double(), C.c_double(), C.c_double()
    lib().oracle_mix_eos(n, *[_dp(a) for a in arr], V, rho, C.byref(p), C.byref(P), C.byref(cs))
    return p.value, P.value, cs.value


def q_of_du(rho, cs, du, c1, c2):
    return lib().oracle_q_of_du(rho, cs, du, c1, c2)


def dt_cell(cfl, l2, v2, cs, du=0.0, c1=0.25, c2=2.0):
    """c.5 candidate with the viscous signal speed of reading DT-Q (du < 0 compresses)."""
    return lib().oracle_dt_cell(cfl, l2, v2, cs, du, c1, c2)


def hg_modes(U):
    """Reading HG: mode amplitudes g[4, 3] of the 8 hex-corner velocities U[8, 3]."""
    U = np.ascontiguousarray(U, dtype=np.float64).reshape(8, 3)
    g = np.zeros((4, 3))
    lib().oracle_hg_modes(_dp(U), _dp(g))
    return g


def hg_corner(g, nu, h):
    g = np.ascontiguousarray(g, dtype=np.float64).reshape(4, 3)
    f = np.zeros(3)
    lib().oracle_hg_corner(_dp(g), nu, int(h), _dp(f))
    return f


def hg_nu(hg, m, cs, Lsum, dt):
    return lib().oracle_hg_nu(hg, m, cs, Lsum, dt)


def swept_volume(PT, PL):
    PT = np.ascontiguousarray(PT, dtype=np.float64).reshape(4, 3)
    PL = np.ascontiguousarray(PL, dtype=np.float64).reshape(4, 3)
    return lib().oracle_swept_volume(_dp(PT), _dp(PL))


def cell_energy(N0, U0, U1, sigma, m, e, dt, nu=0.0):
    N0 = np.ascontiguousarray(N0, dtype=np.float64).reshape(8, 3)
    U0 = np.ascontiguousarray(U0, dtype=np.float64).reshape(8, 3)
    U1 = np.ascontiguousarray(U1, dtype=np.float64).reshape(8, 3)
    return lib().oracle_cell_energy(_dp(N0), _dp(U0), _dp(U1), sigma, nu, m, e, dt)
