"""CPU checks of the C-ABI library: it builds for sm_100a, loads, and exports every declared symbol."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hdgb.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hdgb_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2007_11891_b200.build import build

    return build()


def test_header_declares_the_hot_path_entry_points():
    names = _declared()
    for must in ("hdgb_ctx_create", "hdgb_op_apply", "hdgb_prec_apply", "hdgb_pcg", "hdgb_face_transform",
                 "hdgb_vec_dot", "hdgb_halo_pack"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header(lib_path):
    from paper_2007_11891_b200 import _lib

    assert set(_declared()) == set(_lib.SIGNATURES)
    L = _lib.lib()
    assert L.hdgb_version().startswith(b"hdgb")
    assert L.hdgb_dot_scratch_doubles() > 0


def test_library_is_sm100a_code(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_ctx_create_rejects_bad_arguments_without_gpu(lib_path):
    from paper_2007_11891_b200 import _lib

    L = _lib.lib()
    d = _lib.Desc()
    d.p = 0  # invalid degree: rejected before any CUDA call
    h = ctypes.c_void_p()
    rc = L.hdgb_ctx_create(ctypes.byref(d), ctypes.byref(h))
    assert rc == _lib.EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without the built library the hot path raises instead of computing."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_2007_11891_b200 import _lib\n"
        "try:\n"
        "    _lib.lib()\n"
        "except _lib.LibraryMissing as e:\n"
        "    print('raised', e)\n"
        "else:\n"
        "    print('loaded')\n" % ROOT)
    env = dict(os.environ, HDGB_LIB=str(tmp_path / "absent.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("raised"), out.stdout
