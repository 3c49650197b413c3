"""C-ABI library checks that need no GPU (-m "not gpu"): the in-tree libstk.so
builds for sm_100a, loads, exports every symbol include/stk.h declares, and
rejects invalid configurations before touching the device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stk.h")


def _lib_path():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_stk_build", os.path.join(ROOT, "paper_1604_07994_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    return b.build()


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:stk_status|int64_t|const char\*)\s+(stk_\w+)\(", src, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("stk_create", "stk_set_viscosity", "stk_assemble", "stk_apply", "stk_smooth",
                 "stk_restrict", "stk_prolong_add", "stk_vcycle", "stk_solve", "stk_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib_path())
    for name in _declared():
        assert hasattr(lib, name), name


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tma_for_the_tiled_kernels():
    out = subprocess.run(["cuobjdump", "-sass", _lib_path()], capture_output=True, text=True).stdout
    assert "UTMALDG" in out          # cp.async.bulk.tensor (TMA) loads


def test_create_rejects_bad_config_without_device():
    lib = ctypes.CDLL(_lib_path())

    class Cfg(ctypes.Structure):
        _fields_ = [("n", ctypes.c_int32), ("n_coarse", ctypes.c_int32), ("form", ctypes.c_int32),
                    ("face", ctypes.c_int32 * 6), ("delta", ctypes.c_double),
                    ("nu_pre", ctypes.c_int32), ("nu_post", ctypes.c_int32), ("nu_inc", ctypes.c_int32),
                    ("omega", ctypes.c_double), ("ncolors_u", ctypes.c_int32), ("krylov", ctypes.c_int32),
                    ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("stream", ctypes.c_void_p)]

    lib.stk_create.argtypes = [ctypes.POINTER(Cfg), ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    lib.stk_create.restype = ctypes.c_int
    h = ctypes.c_void_p()
    for n, nc, colors, faces in [(12, 4, 2, (0,) * 6), (16, 4, 3, (0,) * 6), (16, 4, 2, (1,) * 6),
                                 (2, 4, 2, (0,) * 6), (16, 32, 2, (0,) * 6)]:
        c = Cfg()
        c.n, c.n_coarse, c.form, c.ncolors_u, c.nranks = n, nc, 0, colors, 1
        for f in range(6):
            c.face[f] = faces[f]
        assert lib.stk_create(ctypes.byref(c), None, ctypes.byref(h)) == -1   # STK_EINVAL


def test_package_refuses_to_import_without_library(tmp_path):
    """No CPU fallback: the binding raises when libstk.so is absent."""
    import shutil
    pkg = tmp_path / "paper_1604_07994_b200"
    shutil.copytree(os.path.join(ROOT, "paper_1604_07994_b200"), pkg,
                    ignore=shutil.ignore_patterns("*.so", "csrc"))
    r = subprocess.run(["python", "-c", "import paper_1604_07994_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr
