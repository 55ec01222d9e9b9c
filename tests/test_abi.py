"""CPU checks of the C-ABI boundary: the library loads, exports exactly what
include/difform_gpu.h declares, and the host-only entry points (no GPU
needed) agree with the reference's semantics."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2404_01249_b200 import _abi as A
from paper_2404_01249_b200 import engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "difform_gpu.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^DFM_API\s+[\w\s\*]+?\b(dfm_\w+)\(", src, flags=re.M)))


def test_header_declares_the_binding_list():
    assert declared() == sorted(engine.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = engine.load_library()
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing


def test_only_the_c_abi_is_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", engine.LIB_PATH], capture_output=True,
                         text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert syms == set(declared())


def test_abi_version_and_defaults():
    lib = engine.load_library()
    assert lib.dfm_abi_version() == 1
    c = A.dfm_config()
    lib.dfm_config_defaults(C.byref(c))
    ref = A.RegistrationConfig()
    for name, _ in A.dfm_config._fields_:
        assert getattr(c, name) == pytest.approx(float(getattr(ref, name))), name


def test_grid_validation_matches_reference_rules():
    lib = engine.load_library()
    ok = A.GridMeta.make_3d(4, 5, 6).c()
    assert lib.dfm_validate_grid(C.byref(ok)) == A.DFM_OK
    for bad in (A.GridMeta(3, (1, 5, 6)), A.GridMeta(2, (4, 5, 2)), A.GridMeta(4, (4, 4, 4)),
                A.GridMeta(3, (4, 4, 4), (1.0, 0.0, 1.0))):
        assert lib.dfm_validate_grid(C.byref(bad.c())) == A.DFM_E_INVALID


@pytest.mark.parametrize("dims,f", [((160, 192, 224), 4.0), ((160, 192, 224), 2.0),
                                    ((13, 11, 9), 3.0), ((1024, 1024, 1024), 8.0),
                                    ((17, 12, 1), 2.0)])
def test_downsample_grid_matches_oracle(oracle_port, dims, f):
    lib = engine.load_library()
    nd = 2 if dims[2] == 1 else 3
    g = A.GridMeta(nd, dims).c()
    fac = (C.c_double * 3)(f, f, f)
    out = A.dfm_grid()
    assert lib.dfm_downsample_grid(C.byref(g), fac, C.byref(out)) == 0
    out2 = A.dfm_grid()
    assert oracle_port.t.lib.orc_downsample_grid(C.byref(g), fac, C.byref(out2)) == 0
    assert tuple(out.dims) == tuple(out2.dims)
    assert tuple(out.spacing) == tuple(out2.spacing)


def test_context_without_gpu_fails_loudly():
    if engine.cuda_available():
        pytest.skip("a GPU is present")
    with pytest.raises((A.DeviceError, A.InvalidArgument)):
        engine.Context(0, "f32")


def test_no_oracle_in_product():
    """The product package must not import or link the CPU checkers."""
    pkg = os.path.join(ROOT, "paper_2404_01249_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("no CPU fallback", ""), f
