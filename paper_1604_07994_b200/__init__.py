"""B200-native matrix-free Stokes operator and Uzawa multigrid (arXiv:1604.07994).

Thin Python binding of the C ABI in ``include/stk.h`` (``libstk.so``, built
in-tree by ``paper_1604_07994_b200.build``).  Argument marshalling only: every
step of the operator and solver runs in the library's CUDA kernels.  There is
no CPU fallback — importing this package without the built library raises.

Functions keep the C names (``stk_create``, ``stk_apply``, ...).  The
``StokesContext`` class bundles them for torch device tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("STK_LIBNAME", "libstk.so"))  # in-tree build variants only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_1604_07994_b200/build.py` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

STK_OK, STK_ENOCONV, STK_EINVAL, STK_ENOMEM, STK_ECUDA, STK_ENCCL, STK_ESTATE, STK_EUNSUP = (
    0, 1, -1, -2, -3, -4, -5, -6)
FORMS = {"mod": 0, "sym": 1, "grad": 2}
BLK_A, BLK_BT, BLK_B, BLK_C, BLK_ALL = 1, 2, 4, 8, 15
HOST, DEVICE = 0, 1


class stk_config(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("n_coarse", ctypes.c_int32), ("form", ctypes.c_int32),
                ("face", ctypes.c_int32 * 6), ("delta", ctypes.c_double),
                ("nu_pre", ctypes.c_int32), ("nu_post", ctypes.c_int32), ("nu_inc", ctypes.c_int32),
                ("omega", ctypes.c_double), ("ncolors_u", ctypes.c_int32), ("krylov", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("coarse_mu", ctypes.c_int32)]


class stk_layout_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("nz_local", ctypes.c_int32), ("z0", ctypes.c_int32),
                ("pitch_x", ctypes.c_int64), ("pitch_y", ctypes.c_int64),
                ("field_stride", ctypes.c_int64), ("vec_len", ctypes.c_int64),
                ("n_irregular", ctypes.c_int64), ("n_vertices", ctypes.c_int64)]


class stk_report(ctypes.Structure):
    _fields_ = [("cycles", ctypes.c_int32), ("rho", ctypes.c_double), ("rel_res", ctypes.c_double),
                ("t_total_s", ctypes.c_double), ("res_hist", ctypes.c_double * 256),
                ("t_level_s", ctypes.c_double * 16), ("nan_seen", ctypes.c_int32)]


_P = ctypes.c_void_p
_S = ctypes.c_int
_sigs = {
    "stk_nccl_unique_id": [_P],
    "stk_partition": [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P],
    "stk_create": [ctypes.POINTER(stk_config), _P, ctypes.POINTER(_P)],
    "stk_loopback_create": [ctypes.c_int32, ctypes.POINTER(_P)],
    "stk_create_loopback": [ctypes.POINTER(stk_config), _P, ctypes.POINTER(_P)],
    "stk_loopback_destroy": [_P],
    "stk_export_classes": [_P, ctypes.c_int32, _P, _P],
    "stk_export_codes": [_P, ctypes.c_int32, _P],
    "stk_set_viscosity": [_P, _P, _P, ctypes.c_int32],
    "stk_cube_range": [_P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
    "stk_assemble": [_P],
    "stk_layout": [_P, ctypes.c_int32, ctypes.POINTER(stk_layout_t)],
    "stk_import": [_P, ctypes.c_int32, _P, ctypes.c_int32, _P],
    "stk_export": [_P, ctypes.c_int32, _P, _P, ctypes.c_int32],
    "stk_zero_eliminated": [_P, ctypes.c_int32, _P],
    "stk_set_coarse_solver": [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32],
    "stk_p0_apply": [_P, _P, _P, _P, _P, ctypes.c_double],
    "stk_p0_fluxes": [_P, _P, _P, _P, ctypes.c_double],
    "stk_p0_solve": [_P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, _P],
    "stk_load_vector": [_P, ctypes.c_int32, _P, _P, ctypes.c_int32, _P],
    "stk_apply": [_P, ctypes.c_int32, ctypes.c_uint32, _P, _P],
    "stk_residual": [_P, ctypes.c_int32, _P, _P, _P, _P],
    "stk_smooth": [_P, ctypes.c_int32, _P, _P, ctypes.c_int32],
    "stk_restrict": [_P, ctypes.c_int32, _P, _P],
    "stk_prolong_add": [_P, ctypes.c_int32, _P, _P],
    "stk_vcycle": [_P, _P, _P],
    "stk_solve": [_P, _P, _P, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(stk_report)],
    "stk_gauge": [_P, ctypes.c_int32, _P],
    "stk_norms": [_P, ctypes.c_int32, _P, _P],
    "stk_set_kernel_mode": [_P, ctypes.c_int32],
    "stk_set_fuse_n": [_P, ctypes.c_int32],
    "stk_set_row_n": [_P, ctypes.c_int32],
    "stk_profile_enable": [_P, ctypes.c_int32],
    "stk_profile_reset": [_P],
    "stk_profile_read": [_P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                         ctypes.POINTER(ctypes.c_double)],
    "stk_destroy": [_P],
}
for _name, _args in _sigs.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _S
_lib.stk_last_error.argtypes = [_P]
_lib.stk_last_error.restype = ctypes.c_char_p
_lib.stk_launch_count.argtypes = [_P]
_lib.stk_launch_count.restype = ctypes.c_int64
_lib.stk_fused_level.argtypes = [_P]
_lib.stk_fused_level.restype = ctypes.c_int32
_lib.stk_row_level.argtypes = [_P]
_lib.stk_row_level.restype = ctypes.c_int32

# C names re-exported verbatim
for _name in list(_sigs) + ["stk_last_error", "stk_launch_count", "stk_fused_level", "stk_row_level"]:
    globals()[_name] = getattr(_lib, _name)


class StkError(RuntimeError):
    def __init__(self, call, status, msg):
        super().__init__(f"{call} failed with status {status}: {msg}")
        self.status = status


def _ptr(t):
    """device/host pointer of a torch tensor or numpy array (no copies)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    assert t.is_contiguous()
    return t.data_ptr()


def partition(n, nranks, rank, n_coarse=4):
    """z-slab partition of the level hierarchy (host only; stk_partition): list of
    dicts per level (finest first) with n, z0, nzl, cz0, cz1, replicated, K0, K1."""
    nlev = ctypes.c_int32()
    out = (ctypes.c_int32 * (8 * 16))()
    s = _lib.stk_partition(n, n_coarse, nranks, rank, ctypes.byref(nlev), out)
    if s != STK_OK:
        raise StkError("stk_partition", s, "bad sizes")
    keys = ("n", "z0", "nzl", "cz0", "cz1", "replicated", "K0", "K1")
    return [dict(zip(keys, out[8 * l:8 * l + 8])) for l in range(nlev.value)]


class LoopbackGroup:
    """nranks contexts of one process on one device (stk_loopback_create): run each
    rank's calls in its own thread (ctypes releases the GIL during library calls)."""

    def __init__(self, nranks):
        h = _P()
        s = _lib.stk_loopback_create(nranks, ctypes.byref(h))
        if s != STK_OK:
            raise StkError("stk_loopback_create", s, "")
        self.h, self.nranks = h, nranks

    def close(self):
        if getattr(self, "h", None):
            _lib.stk_loopback_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    s = _lib.stk_nccl_unique_id(buf)
    if s != STK_OK:
        raise StkError("stk_nccl_unique_id", s, "NCCL unavailable")
    return bytes(buf)


class StokesContext:
    """One rank (one GPU) of the distributed operator / solver."""

    def __init__(self, n, form="mod", faces=(0,) * 6, delta=1.0 / 12.0, n_coarse=4,
                 nu_pre=3, nu_post=3, nu_inc=2, omega=0.3, ncolors_u=2, krylov=0, rank=0, nranks=1,
                 stream=None, nccl_id: bytes | None = None, loopback: LoopbackGroup | None = None,
                 coarse_mu="arith"):
        import torch
        self.torch = torch
        cfg = stk_config()
        cfg.n, cfg.n_coarse, cfg.form = n, n_coarse, FORMS[form]
        for f in range(6):
            cfg.face[f] = int(faces[f])
        cfg.delta, cfg.nu_pre, cfg.nu_post, cfg.nu_inc = delta, nu_pre, nu_post, nu_inc
        cfg.omega, cfg.ncolors_u, cfg.rank, cfg.nranks = omega, ncolors_u, rank, nranks
        cfg.krylov = krylov
        cfg.coarse_mu = {"arith": 1, "harmonic": 2}[coarse_mu]
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        cfg.stream = stream.cuda_stream
        self.cfg = cfg
        self.n, self.form, self.faces = n, form, tuple(faces)
        h = _P()
        idbuf = None
        if nccl_id is not None:
            idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        if loopback is not None:
            s = _lib.stk_create_loopback(ctypes.byref(cfg), loopback.h, ctypes.byref(h))
        else:
            s = _lib.stk_create(ctypes.byref(cfg), idbuf, ctypes.byref(h))
        self.h = h
        if s != STK_OK:
            msg = _lib.stk_last_error(h).decode() if h.value else ""
            if h.value:
                _lib.stk_destroy(h)
                self.h = None
            raise StkError("stk_create", s, msg)
        self.nlev = 0
        while True:
            lay = stk_layout_t()
            if _lib.stk_layout(self.h, self.nlev, ctypes.byref(lay)) != STK_OK:
                break
            self.nlev += 1

    # -- plumbing -------------------------------------------------------------
    def _chk(self, call, s, allow=(STK_OK,)):
        if s not in allow:
            raise StkError(call, s, _lib.stk_last_error(self.h).decode())
        return s

    def close(self):
        if getattr(self, "h", None):
            _lib.stk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layout(self, level=0) -> stk_layout_t:
        lay = stk_layout_t()
        self._chk("stk_layout", _lib.stk_layout(self.h, level, ctypes.byref(lay)))
        return lay

    def cube_range(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        self._chk("stk_cube_range", _lib.stk_cube_range(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def partition(self):
        return partition(self.n, self.cfg.nranks, self.cfg.rank, self.cfg.n_coarse)

    def export_classes(self, level=0):
        """(classes uint8 [stored cube layers][n][n][6], emu (.., 2) float64) of a level."""
        p = self.partition()[level]
        m = p["n"]
        cnt = (p["cz1"] - p["cz0"]) * m * m * 6
        cls = np.empty(cnt, dtype=np.uint8)
        emu = np.empty((cnt, 2), dtype=np.float64)
        self._chk("stk_export_classes", _lib.stk_export_classes(self.h, level, _ptr(cls), _ptr(emu)))
        return cls, emu

    def export_codes(self, level=0):
        lay = self.layout(level)
        out = np.empty(lay.n_vertices, dtype=np.uint8)
        self._chk("stk_export_codes", _lib.stk_export_codes(self.h, level, _ptr(out)))
        return out

    def new_vector(self, level=0):
        return self.torch.zeros(self.layout(level).vec_len, dtype=self.torch.float64, device="cuda")

    # -- setup ----------------------------------------------------------------
    def set_viscosity(self, elem_class: np.ndarray, class_mu):
        ec = np.ascontiguousarray(elem_class, dtype=np.uint8)
        mu = np.ascontiguousarray(class_mu, dtype=np.float64)
        self._chk("stk_set_viscosity", _lib.stk_set_viscosity(self.h, _ptr(ec), _ptr(mu), len(mu)))

    def assemble(self):
        self._chk("stk_assemble", _lib.stk_assemble(self.h))

    def p0_apply(self, x, p0, y=None, y0=None, gamma=1.0):
        """Stabilised P1-P0 operator: y = A u + B0^T p0 (level-0
        vector), y0 = B0 u - C0 p0 (6 n^3 per-tet pressures, device tensor)."""
        y = self.new_vector(0) if y is None else y
        p0 = p0.contiguous()
        y0 = self.torch.empty_like(p0) if y0 is None else y0
        self._chk("stk_p0_apply", _lib.stk_p0_apply(self.h, _ptr(x), _ptr(p0), _ptr(y), _ptr(y0), gamma))
        return y, y0

    def p0_solve(self, b, b0, x=None, x0=None, gamma=1.0, rtol=1e-8, max_its=300, m=30):
        """P1-P0 solve (stk_p0_solve): returns (x level vector, x0 per-tet tensor, report)."""
        x = self.new_vector(0) if x is None else x
        b0 = b0.contiguous()
        x0 = self.torch.zeros_like(b0) if x0 is None else x0
        rep = stk_report()
        s = _lib.stk_p0_solve(self.h, _ptr(b), _ptr(b0), _ptr(x), _ptr(x0), gamma, rtol, max_its, m,
                              ctypes.byref(rep))
        self._chk("stk_p0_solve", s, allow=(STK_OK, STK_ENOCONV))
        return x, x0, rep

    def p0_fluxes(self, x, p0, gamma=1.0):
        """P1-P0 local flux post-process: (6 n^3, 4) facet fluxes."""
        p0 = p0.contiguous()
        fl = self.torch.empty((p0.numel(), 4), dtype=self.torch.float64, device=p0.device)
        self._chk("stk_p0_fluxes", _lib.stk_p0_fluxes(self.h, _ptr(x), _ptr(p0), _ptr(fl), gamma))
        return fl

    def set_coarse_solver(self, kind="direct", minres_its=20, cg_its=4):
        """Coarsest-level solver: "direct" (dense inverse of the A_tr system) or "minres"
        (the paper's A_sym + corrected right-hand side + preconditioned MINRES,
        P:1245-1298); re-assembles."""
        k = {"direct": 0, "minres": 1}[kind]
        self._chk("stk_set_coarse_solver", _lib.stk_set_coarse_solver(self.h, k, minres_its, cg_its))
        self.assemble()

    def set_kernel_mode(self, mode: int):
        self._chk("stk_set_kernel_mode", _lib.stk_set_kernel_mode(self.h, mode))

    def set_fuse_n(self, fuse_n: int):
        """Levels with n_l <= fuse_n run the V-cycle in one persistent kernel (0: off)."""
        self._chk("stk_set_fuse_n", _lib.stk_set_fuse_n(self.h, fuse_n))

    def set_row_n(self, row_n: int):
        """V-cycle levels >= 1 with n_l <= row_n run the one-thread-per-row kernels (0: off)."""
        self._chk("stk_set_row_n", _lib.stk_set_row_n(self.h, row_n))

    def row_level(self) -> int:
        return _lib.stk_row_level(self.h)

    def fused_level(self) -> int:
        return _lib.stk_fused_level(self.h)

    def launch_count(self) -> int:
        return _lib.stk_launch_count(self.h)

    PROFILE_OPS = ("apply", "residual", "vel_pass", "p_pass1", "p_pass2", "restrict", "prolong",
                   "coarse", "reduce", "krylov", "coarse_graph", "fused", "vel_repeat", "fwd_sweep")

    def profile(self, on=True):
        """Event-time every launch: True/1 (the coarse-level CUDA graph timed as one
        op, 'coarse_graph'), 2 (every launch, graph disabled), False/0 off."""
        self._chk("stk_profile_enable", _lib.stk_profile_enable(self.h, int(on)))

    def profile_reset(self):
        self._chk("stk_profile_reset", _lib.stk_profile_reset(self.h))

    def profile_read(self, op, level=-1):
        """(launches, total ms) of one op ('vel_pass', ...) on a level (-1 = all)."""
        q = self.PROFILE_OPS.index(op) if isinstance(op, str) else op
        n, ms = ctypes.c_int64(), ctypes.c_double()
        self._chk("stk_profile_read", _lib.stk_profile_read(self.h, q, level, ctypes.byref(n), ctypes.byref(ms)))
        return n.value, ms.value

    # -- vectors --------------------------------------------------------------
    def import_(self, canon, level=0, out=None, mask=True):
        """canonical (4, owned vertices) host numpy or device tensor -> padded device vector;
        mask: eliminated velocity DoFs set to 0 (operator inputs; False for a nodal forcing)."""
        out = self.new_vector(level) if out is None else out
        if isinstance(canon, np.ndarray):
            c = np.ascontiguousarray(canon, dtype=np.float64)
            self._chk("stk_import", _lib.stk_import(self.h, level, _ptr(c), HOST, _ptr(out)))
        else:
            c = canon.contiguous()
            self._chk("stk_import", _lib.stk_import(self.h, level, _ptr(c), DEVICE, _ptr(out)))
        if mask:
            self._chk("stk_zero_eliminated", _lib.stk_zero_eliminated(self.h, level, _ptr(out)))
        return out

    def export(self, vec, level=0) -> np.ndarray:
        lay = self.layout(level)
        out = np.empty((4, lay.n_vertices), dtype=np.float64)
        self._chk("stk_export", _lib.stk_export(self.h, level, _ptr(vec), _ptr(out), HOST))
        return out

    def export_device(self, vec, level=0, out=None):
        lay = self.layout(level)
        out = self.torch.empty((4, lay.n_vertices), dtype=self.torch.float64, device="cuda") if out is None else out
        self._chk("stk_export", _lib.stk_export(self.h, level, _ptr(vec), _ptr(out), DEVICE))
        return out

    def load_nodal(self, f_canon, b=None):
        """b = (M f, 0) for nodal forcing f (3, owned vertices)."""
        lay = self.layout(0)
        f4 = np.zeros((4, lay.n_vertices)) if isinstance(f_canon, np.ndarray) else None
        if f4 is not None:
            f4[:3] = f_canon
            fv = self.import_(f4, mask=False)
        else:
            t = self.torch.zeros((4, lay.n_vertices), dtype=self.torch.float64, device="cuda")
            t[:3] = f_canon
            fv = self.import_(t, mask=False)
        b = self.new_vector(0) if b is None else b
        self._chk("stk_load_vector", _lib.stk_load_vector(self.h, 0, _ptr(fv), None, 0, _ptr(b)))
        return b

    def load_element(self, f_cls: np.ndarray, table, b=None):
        fc = self.torch.from_numpy(np.ascontiguousarray(f_cls, dtype=np.uint8)).cuda()
        tab = np.ascontiguousarray(table, dtype=np.float64).reshape(-1)
        b = self.new_vector(0) if b is None else b
        self._chk("stk_load_vector", _lib.stk_load_vector(self.h, 1, _ptr(fc), _ptr(tab),
                                                          len(tab) // 3, _ptr(b)))
        self.torch.cuda.current_stream().synchronize()
        return b

    # -- operator / solver ------------------------------------------------------
    def apply(self, x, y=None, level=0, blocks=BLK_ALL):
        y = self.new_vector(level) if y is None else y
        self._chk("stk_apply", _lib.stk_apply(self.h, level, blocks, _ptr(x), _ptr(y)))
        return y

    def residual(self, x, b, r=None, level=0, norms=False):
        r = self.new_vector(level) if r is None else r
        nb = np.zeros(5) if norms else None
        self._chk("stk_residual", _lib.stk_residual(self.h, level, _ptr(x), _ptr(b), _ptr(r), _ptr(nb)))
        return (r, nb) if norms else r

    def norms(self, x, level=0):
        out = np.zeros(5)
        self._chk("stk_norms", _lib.stk_norms(self.h, level, _ptr(x), _ptr(out)))
        return out

    def smooth(self, x, b, steps=1, level=0):
        self._chk("stk_smooth", _lib.stk_smooth(self.h, level, _ptr(x), _ptr(b), steps))
        return x

    def restrict(self, r_f, b_c=None, fine_level=0):
        b_c = self.new_vector(fine_level + 1) if b_c is None else b_c
        self._chk("stk_restrict", _lib.stk_restrict(self.h, fine_level, _ptr(r_f), _ptr(b_c)))
        return b_c

    def prolong_add(self, x_c, x_f, coarse_level=1):
        self._chk("stk_prolong_add", _lib.stk_prolong_add(self.h, coarse_level, _ptr(x_c), _ptr(x_f)))
        return x_f

    def vcycle(self, b, x):
        self._chk("stk_vcycle", _lib.stk_vcycle(self.h, _ptr(b), _ptr(x)))
        return x

    def gauge(self, x, level=0):
        self._chk("stk_gauge", _lib.stk_gauge(self.h, level, _ptr(x)))
        return x

    def solve(self, b, x=None, rtol=1e-8, max_cycles=100, raise_on_noconv=False):
        x = self.new_vector(0) if x is None else x
        rep = stk_report()
        s = _lib.stk_solve(self.h, _ptr(b), _ptr(x), rtol, max_cycles, ctypes.byref(rep))
        self._chk("stk_solve", s, allow=(STK_OK,) if raise_on_noconv else (STK_OK, STK_ENOCONV))
        return x, rep
