"""Thin Python binding of libsale (include/sale.h): argument marshalling only.

Every step of the SALE cycle runs in libsale's CUDA kernels; PyTorch supplies
the device workspace, the stream and (for multi-GPU) the process group that
broadcasts the NCCL unique id.  There is no CPU fallback: if libsale.so is
missing or no GPU is present, constructing a context raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SALE_LIB_PATH") or os.path.join(_HERE, "lib", "libsale.so")  # override: experiments only

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ETANGLED, EDTCOLLAPSE, ENEGMASS, EPOISONED, EREPLICA = range(10)
CODE_NAMES = ["OK", "EINVAL", "ENOMEM", "ECUDA", "ENCCL", "ETANGLED", "EDTCOLLAPSE", "ENEGMASS",
              "EPOISONED", "EREPLICA"]
LAGRANGE, EULER = 0, 1
FIELDS = {"X": 0, "Y": 1, "Z": 2, "UX": 3, "UY": 4, "UZ": 5, "NODE_MASS": 6,
          "MASS": 7, "E": 8, "RHO": 9, "VOL": 10, "P": 11, "Q": 12, "CS": 13}
MAX_MAT = 4
HALO_COPY, HALO_PEER = 0, 1  # sale_params.halo
for _m in range(MAX_MAT):  # material fields (nmat >= 1): volume fraction, mass, specific energy
    FIELDS[f"MAT_F{_m}"], FIELDS[f"MAT_M{_m}"], FIELDS[f"MAT_E{_m}"] = 16 + _m, 20 + _m, 24 + _m
NODE_FIELDS = ("X", "Y", "Z", "UX", "UY", "UZ", "NODE_MASS")
EXPORTS = ("sale_workspace_bytes", "sale_nccl_unique_id", "sale_create", "sale_step",
           "sale_step_async", "sale_sync", "sale_get_field", "sale_set_field", "sale_get_clock",
           "sale_set_clock", "sale_get_layout", "sale_kernel_launches", "sale_profile_enable",
           "sale_profile_read", "sale_halo_plan", "sale_local_layout", "sale_steinberg",
           "sale_last_error", "sale_destroy")
K_CLASSES = ("begin", "prologue", "lagrange", "remap", "halo")


class SaleParams(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32),
                ("nz", C.c_int32), ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("gamma", C.c_double), ("q_lin", C.c_double), ("q_quad", C.c_double),
                ("cfl", C.c_double), ("dt_growth", C.c_double), ("t_end", C.c_double),
                ("rezone", C.c_int32), ("reflect_mask", C.c_uint32), ("rho0", C.c_double),
                ("e_background", C.c_double), ("e_deposit", C.c_double), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_uint64),
                ("device", C.c_int32), ("overlap", C.c_int32), ("local_slabs", C.c_int32),
                ("nmat", C.c_int32), ("mat_gamma", C.c_double * MAX_MAT), ("hg", C.c_double),
                ("halo", C.c_int32)]


class SaleSteinberg(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("G0", "GP", "GT", "Y0", "Ymax", "beta", "n", "cv", "rho0", "T0")]


class SaleHaloMsg(C.Structure):
    _fields_ = [("peer", C.c_int32), ("send", C.c_int32), ("field", C.c_int32),
                ("first_plane", C.c_int32), ("offset", C.c_int64), ("count", C.c_int64)]


class SaleError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {CODE_NAMES[code] if 0 <= code < len(CODE_NAMES) else code}")


_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load libsale.so (build it with paper_2209_01983_b200.build.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libsale.so not built ({LIB_PATH}); run __graft_entry__.build()")
            L = C.CDLL(LIB_PATH)
            P, vp = C.POINTER, C.c_void_p
            d, i32, i64, u64 = C.c_double, C.c_int32, C.c_int64, C.c_uint64
            L.sale_workspace_bytes.argtypes = [P(SaleParams)]
            L.sale_workspace_bytes.restype = u64
            L.sale_nccl_unique_id.argtypes = [vp]
            L.sale_nccl_unique_id.restype = i32
            L.sale_create.argtypes = [P(SaleParams), P(vp)]
            L.sale_create.restype = i32
            L.sale_step.argtypes = [vp, i32, P(i32)]
            L.sale_step.restype = i32
            L.sale_step_async.argtypes = [vp, i32]
            L.sale_step_async.restype = i32
            L.sale_sync.argtypes = [vp, P(i32)]
            L.sale_sync.restype = i32
            L.sale_get_field.argtypes = [vp, i32, vp, u64, i32]
            L.sale_get_field.restype = i32
            L.sale_set_field.argtypes = [vp, i32, vp, u64, i32]
            L.sale_set_field.restype = i32
            L.sale_get_clock.argtypes = [vp, P(d), P(d), P(i64), P(i32)]
            L.sale_get_clock.restype = i32
            L.sale_set_clock.argtypes = [vp, d, d, i64]
            L.sale_set_clock.restype = i32
            L.sale_get_layout.argtypes = [vp, P(i32), P(i32)]
            L.sale_get_layout.restype = i32
            L.sale_kernel_launches.argtypes = [vp]
            L.sale_kernel_launches.restype = i64
            L.sale_profile_enable.argtypes = [vp, i32]
            L.sale_profile_enable.restype = i32
            L.sale_profile_read.argtypes = [vp, i32, P(d), P(i64)]
            L.sale_profile_read.restype = i32
            L.sale_halo_plan.argtypes = [P(SaleParams), i32, P(SaleHaloMsg), i32]
            L.sale_halo_plan.restype = i32
            L.sale_local_layout.argtypes = [P(SaleParams), P(i32), P(i32), P(i32), P(i32), P(i32)]
            L.sale_local_layout.restype = i32
            L.sale_steinberg.argtypes = [vp, P(SaleSteinberg), vp, vp, vp, u64]
            L.sale_steinberg.restype = i32
            L.sale_last_error.argtypes = [vp]
            L.sale_last_error.restype = C.c_char_p
            L.sale_destroy.argtypes = [vp]
            L.sale_destroy.restype = None
            _lib = L
    return _lib


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().sale_nccl_unique_id(buf)
    if rc:
        raise SaleError(rc, "sale_nccl_unique_id")
    return buf.raw


def make_params(cfg: dict, *, rank=0, nranks=1, device=0, local_slabs=1) -> SaleParams:
    p = SaleParams()
    p.abi_version = 4
    for k in ("nx", "ny", "nz", "lx", "ly", "lz", "gamma", "q_lin", "q_quad", "cfl", "dt_growth",
              "t_end", "rezone", "reflect_mask", "rho0", "e_background", "e_deposit"):
        setattr(p, k, cfg[k])
    p.rank, p.nranks, p.device = rank, nranks, device
    p.local_slabs = local_slabs
    p.hg = float(cfg.get("hg", 0.0))
    p.overlap = int(cfg.get("overlap", 0))
    p.halo = int(cfg.get("halo", HALO_COPY))
    gam = list(cfg.get("mat_gamma", ()))[:MAX_MAT]  # nmat > MAX_MAT is rejected by libsale
    p.nmat = int(cfg.get("nmat", 0))
    p.mat_gamma = (C.c_double * MAX_MAT)(*(gam + [0.0] * (MAX_MAT - len(gam))))
    return p


FIELD_NAMES = {v: k for k, v in FIELDS.items()}


def halo_plan(cfg: dict, rank: int, nranks: int, full: bool = False) -> list[dict]:
    """The X1 message plan of one rank (host-only; what sale_step sends via NCCL)."""
    p = make_params(cfg, rank=rank, nranks=nranks)
    n = lib().sale_halo_plan(C.byref(p), 1 if full else 0, None, 0)
    if n < 0:
        raise SaleError(EINVAL, "sale_halo_plan")
    buf = (SaleHaloMsg * max(n, 1))()
    lib().sale_halo_plan(C.byref(p), 1 if full else 0, buf, n)
    return [{"peer": m.peer, "send": bool(m.send), "field": FIELD_NAMES[m.field],
             "first_plane": m.first_plane, "offset": m.offset, "count": m.count} for m in buf[:n]]


def local_layout(cfg: dict, rank: int, nranks: int) -> dict:
    p = make_params(cfg, rank=rank, nranks=nranks)
    k0, k1, g, nn, nc = (C.c_int32() for _ in range(5))
    rc = lib().sale_local_layout(C.byref(p), C.byref(k0), C.byref(k1), C.byref(g), C.byref(nn), C.byref(nc))
    if rc:
        raise SaleError(rc, "sale_local_layout")
    return {"k0": k0.value, "k1": k1.value, "ghost": g.value, "node_planes": nn.value,
            "cell_planes": nc.value}


def workspace_bytes(cfg: dict, **kw) -> int:
    return int(lib().sale_workspace_bytes(C.byref(make_params(cfg, **kw))))


class Sale:
    """One libsale context on one GPU (one z-slab of the mesh per rank).

    cfg: the sale_params values (configs.config / configs.sedov ...); optional
    cfg["nmat"] (1..4) and cfg["mat_gamma"] add the material axis (fields MAT_F<k>,
    MAT_M<k>, MAT_E<k>; include/sale.h); cfg["hg"] the hourglass coefficient (0 if
    absent); cfg["overlap"] the boundary-first mode (0 automatic, 1 on, -1 off); cfg["halo"]
    HALO_COPY (0, default) or HALO_PEER (1: the producing kernels store the ghost planes
    straight into the neighbours').  local_slabs > 1 splits the mesh into emulated ranks on one GPU."""

    def __init__(self, cfg: dict, *, device: int = 0, stream=None, rank: int = 0, nranks: int = 1,
                 nccl_id: bytes | None = None, local_slabs: int = 1):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libsale needs a CUDA device (no CPU fallback)")
        L = lib()
        self.cfg = dict(cfg)
        self._L = L
        p = make_params(cfg, rank=rank, nranks=nranks, device=device, local_slabs=local_slabs)
        nbytes = L.sale_workspace_bytes(C.byref(p))
        if nbytes == 0:
            raise SaleError(EINVAL, "sale_workspace_bytes")
        self.torch_device = torch.device("cuda", device)
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.torch_device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.torch_device)
        p.workspace = self.workspace.data_ptr()
        p.workspace_bytes = nbytes
        p.stream = self.stream.cuda_stream
        self._id = None
        if nccl_id is not None:
            self._id = C.create_string_buffer(nccl_id, 128)
            p.nccl_unique_id = C.cast(self._id, C.c_void_p)
        self._p = p
        h = C.c_void_p()
        rc = L.sale_create(C.byref(p), C.byref(h))
        if rc:
            raise SaleError(rc, "sale_create")
        self._h = h
        k0, k1 = C.c_int32(), C.c_int32()
        L.sale_get_layout(h, C.byref(k0), C.byref(k1))
        self.k0, self.k1 = k0.value, k1.value
        nx, ny = cfg["nx"], cfg["ny"]
        self.node_shape = (self.k1 - self.k0 + 1, ny + 1, nx + 1)
        self.cell_shape = (self.k1 - self.k0, ny, nx)

    def close(self):
        if getattr(self, "_h", None):
            self._L.sale_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- stepping ---------------------------------------------------------
    def step(self, n: int):
        """Run n cycles (synchronous).  Returns (status code, cycles done)."""
        done = C.c_int32(0)
        rc = self._L.sale_step(self._h, int(n), C.byref(done))
        return rc, done.value

    def step_async(self, n: int) -> None:
        rc = self._L.sale_step_async(self._h, int(n))
        if rc:
            raise SaleError(rc, "sale_step_async: " + self.last_error())

    def sync(self):
        done = C.c_int32(0)
        rc = self._L.sale_sync(self._h, C.byref(done))
        return rc, done.value

    # ---- fields -----------------------------------------------------------
    def get(self, field: str, out=None):
        """Owned slab of a field: numpy (host) by default, or into `out` (a
        contiguous float64 torch tensor on this device)."""
        shape = self.node_shape if field in NODE_FIELDS else self.cell_shape
        if out is None:
            arr = np.empty(shape, dtype=np.float64)
            rc = self._L.sale_get_field(self._h, FIELDS[field], arr.ctypes.data, arr.size, 0)
        else:
            arr = out
            rc = self._L.sale_get_field(self._h, FIELDS[field], out.data_ptr(), out.numel(),
                                        1 if out.is_cuda else 0)
        if rc:
            raise SaleError(rc, f"sale_get_field({field}): " + self.last_error())
        return arr

    def steinberg(self, params, eps_p=None, out=None):
        """Steinberg shear modulus and yield stress of the owned cells (Fig. 6b;
        include/sale.h sale_steinberg).  params: one dict, or with a material axis a
        list of nmat dicts (outputs then gain a leading material axis).  eps_p: plastic
        strain (array of the cell shape) or None.  Returns (shear, yield) as float64
        device tensors (or fills the pair `out`)."""
        import torch
        plist = list(params) if isinstance(params, (list, tuple)) else [params]
        if len(plist) != max(int(self.cfg.get("nmat", 0)), 1):
            raise ValueError("sale_steinberg needs one parameter set per material")
        arr = (SaleSteinberg * len(plist))(*[SaleSteinberg(*[float(d[n]) for n, _ in SaleSteinberg._fields_])
                                             for d in plist])
        shape = ((len(plist),) + self.cell_shape) if isinstance(params, (list, tuple)) else self.cell_shape
        sh, y = out if out is not None else (torch.empty(shape, dtype=torch.float64, device=self.torch_device),
                                             torch.empty(shape, dtype=torch.float64, device=self.torch_device))
        sp = arr
        ep = None
        if eps_p is not None:
            ep = torch.as_tensor(np.ascontiguousarray(eps_p, dtype=np.float64)).to(self.torch_device) \
                if not hasattr(eps_p, "data_ptr") else eps_p
        rc = self._L.sale_steinberg(self._h, C.cast(sp, C.POINTER(SaleSteinberg)), None if ep is None else ep.data_ptr(),
                                    sh.data_ptr(), y.data_ptr(), sh.numel() // len(plist))
        if rc:
            raise SaleError(rc, "sale_steinberg: " + self.last_error())
        return sh, y

    def set(self, field: str, arr) -> None:
        if hasattr(arr, "data_ptr"):  # torch tensor: device, or (pinned) host memory
            rc = self._L.sale_set_field(self._h, FIELDS[field], arr.data_ptr(), arr.numel(),
                                        1 if arr.is_cuda else 0)
        else:
            a = np.ascontiguousarray(arr, dtype=np.float64)
            rc = self._L.sale_set_field(self._h, FIELDS[field], a.ctypes.data, a.size, 0)
        if rc:
            raise SaleError(rc, f"sale_set_field({field}): " + self.last_error())

    def clock(self) -> dict:
        t, dt, cyc, fin = C.c_double(), C.c_double(), C.c_int64(), C.c_int32()
        rc = self._L.sale_get_clock(self._h, C.byref(t), C.byref(dt), C.byref(cyc), C.byref(fin))
        if rc:
            raise SaleError(rc, "sale_get_clock")
        return {"t": t.value, "dt_last": dt.value, "cycle": cyc.value, "finished": fin.value}

    def set_clock(self, t: float, dt_last: float, cycle: int) -> None:
        rc = self._L.sale_set_clock(self._h, t, dt_last, cycle)
        if rc:
            raise SaleError(rc, "sale_set_clock")

    def launches(self) -> int:
        return int(self._L.sale_kernel_launches(self._h))

    def profile(self, on: bool) -> None:
        """Enable (and reset) / disable per-kernel-class CUDA-event timing."""
        self._L.sale_profile_enable(self._h, 1 if on else 0)

    def profile_read(self) -> dict:
        """{class: (total device ms, timed launch groups)} since profile(True)."""
        out = {}
        for k, name in enumerate(K_CLASSES):
            ms, n = C.c_double(), C.c_int64()
            self._L.sale_profile_read(self._h, k, C.byref(ms), C.byref(n))
            out[name] = (ms.value, n.value)
        return out

    def last_error(self) -> str:
        return self._L.sale_last_error(self._h).decode()
