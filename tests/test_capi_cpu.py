"""C-ABI library checks that need no GPU: the in-tree .so loads and exports
every symbol include/taudg.h declares; the ctypes struct layouts match the
header; the product fails loudly (DeviceError) without a device."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "taudg.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(tdg_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1806_11456_b200 import _lib, build

    build.build(verbose=False)
    lib = C.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    # and the Python binding declares a signature for each of them
    assert set(names) <= set(_lib.SIGNATURES)


def test_struct_fields_follow_header_order():
    from paper_1806_11456_b200 import _lib

    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for struct, cls in (("tdg_plan_desc", _lib.PlanDesc), ("tdg_transfer_desc", _lib.TransferDesc)):
        end = text.index("} " + struct + ";")
        body = text[text.rindex("typedef struct {", 0, end) + len("typedef struct {"): end]
        fields = [re.sub(r"\[.*\]", "", decl.split()[-1]).lstrip("*")
                  for decl in body.split(";") if decl.strip()]
        assert [f for f, _ in cls._fields_] == fields, struct


def test_version_and_error_strings():
    from paper_1806_11456_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.tdg_version()
    assert lib.tdg_plan_destroy(None) == 0
    assert lib.tdg_apply(None, None, None, 0, None) == 5      # TDG_E_ARG
    assert b"null" in lib.tdg_last_error()


def test_no_cpu_fallback_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_1806_11456_b200 import errors, fields, mesh, operators, physics

    msh = mesh.build_box(2, 2, 1)
    law = physics.NavierStokes()
    with pytest.raises(errors.DeviceError):
        operators.DGOperator(msh, law, fields.OrderField.uniform(4, 2))


def test_spectral_tables_layout():
    from paper_1806_11456_b200 import spectral

    for fam in ("LG", "LGL"):
        t = spectral.device_tables(fam)
        assert len(t) == spectral.TABLES_LEN == 4800
        n = 5
        dh = t[spectral.OFF_DHAT + n * 64: spectral.OFF_DHAT + (n + 1) * 64].reshape(8, 8)[: n + 1, : n + 1]
        x, w = spectral.rule(n, fam)
        assert np.allclose(dh, w[:, None] * spectral.dmat(n, fam))
        T = t[spectral.OFF_T + (4 * 8 + 6) * 64: spectral.OFF_T + (4 * 8 + 6) * 64 + 64].reshape(8, 8)
        assert np.allclose(T[:7, :5], spectral.transfer(4, 6, fam))
