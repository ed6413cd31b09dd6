"""CPU-side checks of the boundary: liblor_b200.so loads and exports every symbol include/lor.h
declares; the binding refuses to run without a GPU (no CPU fallback); the product package never
imports the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "lor.h")
PKG = os.path.join(ROOT, "paper_2210_12253_b200")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lor_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2210_12253_b200 import build
    return build.build(verbose=False)


def test_header_declares_the_survey_entry_points():
    syms = declared_symbols()
    for s in ("lor_setup", "lor_destroy", "lor_sync", "lor_query", "lor_query_discrete", "lor_assemble_h1",
              "lor_assemble_nd", "lor_assemble_rt", "lor_discrete_grad", "lor_discrete_curl", "lor_dof_map",
              "lor_nccl_get_unique_id"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_setup_rejects_bad_arguments_without_touching_the_gpu(libpath):
    from paper_2210_12253_b200.lor import _SetupArgs, lib
    L = lib()
    h = ctypes.c_void_p()
    a = _SetupArgs()
    a.dim = 4  # invalid
    assert L.lor_setup(ctypes.byref(a), ctypes.byref(h)) == 1
    assert L.lor_setup(None, ctypes.byref(h)) == 1


def test_no_cpu_fallback():
    import torch
    from paper_2210_12253_b200 import meshgen as mg
    from paper_2210_12253_b200.lor import LOR, LorError
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(LorError):
        LOR(mg.box_mesh(3, (1, 1, 1), 2))


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|lor_oracle|liblor_oracle", txt, re.M), f


def test_setup_error_message_without_context():
    """lor_setup has no context to hold its message: lor_last_error(NULL) returns it (boundary
    defect of round 1: the binding printed 'see stderr' with nothing on stderr)."""
    import ctypes
    from paper_2210_12253_b200 import meshgen as mg
    from paper_2210_12253_b200.lor import _SetupArgs, lib
    L = lib()
    m = mg.box_mesh(3, (2, 2, 2), 2)
    vert = np.ascontiguousarray(m.vert)
    elem = np.ascontiguousarray(m.elem, dtype=np.int64)
    a = _SetupArgs()
    a.dim, a.p = 3, 9
    a.n_vert, a.vert_xyz = vert.shape[0], vert.ctypes.data
    a.n_elem, a.elem_vert = elem.shape[0], elem.ctypes.data
    a.rank, a.nranks = 0, 1
    h = ctypes.c_void_p()
    assert L.lor_setup(ctypes.byref(a), ctypes.byref(h)) == 1
    msg = L.lor_last_error(None).decode()
    assert "invalid argument" in msg and "p <= 8" in msg
