"""CPU-side checks of the C-ABI boundary: libsvf.so builds, loads, exports every symbol include/svf.h declares,
its svf_params layout matches the header, and it refuses to run without a GPU (there is no CPU path)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "svf.h")


@pytest.fixture(scope="module")
def svflib():
    from paper_2601_08528_b200 import build_lib

    build_lib.build()
    from paper_2601_08528_b200 import _lib

    return _lib


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:svf_status|void|const char\*)\s+(svf_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("svf_build", "svf_search", "svf_insert", "svf_delete", "svf_knn_exact", "svf_merge_topk",
              "svf_export", "svf_import", "svf_link_candidates", "svf_destroy", "svf_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(svflib):
    L = svflib.lib()
    for f in header_functions():
        assert hasattr(L, f), f
    out = subprocess.run(["nm", "-D", "--defined-only", svflib.LIB_PATH], capture_output=True, text=True).stdout
    for f in header_functions():
        assert re.search(rf"\bT {f}$", out, re.M), f
    assert set(svflib.EXPORTED) == set(header_functions())


def test_params_struct_layout_matches_header(svflib, tmp_path):
    prog = tmp_path / "p.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "svf.h"\nint main(){printf("%zu",'
                    'sizeof(svf_params));' + "".join(
                        f'printf(" %zu", offsetof(svf_params, {f}));' for f, _ in svflib.SvfParams._fields_) +
                    "return 0;}\n")
    exe = tmp_path / "p"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == ctypes.sizeof(svflib.SvfParams)
    for (f, _), off in zip(svflib.SvfParams._fields_, vals[1:]):
        assert getattr(svflib.SvfParams, f).offset == off, f


def test_default_params_and_error_paths_without_gpu(svflib):
    L = svflib.lib()
    p = svflib.SvfParams()
    L.svf_default_params(ctypes.byref(p), 128, 64)
    assert (p.dim, p.degree, p.metric, p.search_width, p.insert_itopk, p.protect_prefix, p.insert_batch,
            p.seed_size, p.seed) == (128, 64, 0, 1, 128, -1, 4096, 4096, 42)
    assert L.svf_last_error() is not None
    # NULL index / bad args are rejected with status codes, never exceptions
    assert L.svf_search(None, None, 1, 10, 10, None, None, None) == svflib.SVF_ERR_INVALID
    assert L.svf_destroy(None) == svflib.SVF_OK
    p.capacity = 100
    X = np.zeros((10, 128), np.float32)
    h = ctypes.c_void_p()
    bad = svflib.SvfParams.from_buffer_copy(p)
    bad.degree = 1
    assert L.svf_build(ctypes.byref(bad), X.ctypes.data, 10, None, ctypes.byref(h)) == svflib.SVF_ERR_INVALID
    import torch

    if not torch.cuda.is_available():
        # no device: the library must refuse (no CPU fallback exists)
        st = L.svf_build(ctypes.byref(p), X.ctypes.data, 10, None, ctypes.byref(h))
        assert st == svflib.SVF_ERR_CUDA, st
        assert b"no CUDA device" in L.svf_last_error()


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    import paper_2601_08528_b200._lib as m

    monkeypatch.setattr(m, "_lib", None)
    monkeypatch.setattr(m, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        m.lib()


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2601_08528_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src), f
