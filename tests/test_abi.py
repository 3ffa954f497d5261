"""CPU-side checks of the boundary: libsale.so loads and exports every symbol
include/sale.h declares; the host-only entry points (no GPU needed) validate
parameters and size the workspace; the binding's struct matches the header."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2209_01983_b200 import build, configs, sale

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return sale.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sale.h")).read()
    return sorted(set(re.findall(r"\b(sale_[a-z_0-9]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported(L):
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(sale.EXPORTS) == syms


def test_struct_layout_matches_header(tmp_path):
    """ctypes SaleParams offsets == the C compiler's offsetof for include/sale.h."""
    names = [n for n, _ in sale.SaleParams._fields_]
    prog = "#include <stdio.h>\n#include <stddef.h>\n#include \"sale.h\"\nint main(void){\n"
    prog += "printf(\"%zu\\n\", sizeof(sale_params));\n"
    for n in names:
        prog += f"printf(\"%zu\\n\", offsetof(sale_params, {n}));\n"
    prog += "return 0;}\n"
    src = tmp_path / "off.c"
    src.write_text(prog)
    exe = tmp_path / "off"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert vals[0] == C.sizeof(sale.SaleParams)
    for n, off in zip(names, vals[1:]):
        assert getattr(sale.SaleParams, n).offset == off, n


def test_workspace_bytes_validates(L):
    cfg, _ = configs.config("C0")
    assert sale.workspace_bytes(cfg) > 0
    assert sale.workspace_bytes(dict(cfg, gamma=1.0)) == 0
    assert sale.workspace_bytes(dict(cfg, nx=0)) == 0
    assert sale.workspace_bytes(dict(cfg, rezone=2)) == 0
    assert sale.workspace_bytes(dict(cfg, hg=-1.0)) == 0
    # the material axis: 0..4 materials, every gamma > 1
    assert sale.workspace_bytes(dict(cfg, nmat=4, mat_gamma=[1.4, 1.5, 1.6, 1.7])) > sale.workspace_bytes(cfg)
    assert sale.workspace_bytes(dict(cfg, nmat=5, mat_gamma=[1.4] * 4)) == 0
    assert sale.workspace_bytes(dict(cfg, nmat=2, mat_gamma=[1.4, 0.9])) == 0
    # slabs must own >= g planes: Euler g = 3
    e = configs.sedov((8, 8, 8), configs.EULER)
    assert sale.workspace_bytes(e, local_slabs=2) > 0
    assert sale.workspace_bytes(e, local_slabs=3) == 0
    # nranks > 1 needs an NCCL id in sale_create, but the size query tolerates it
    p = sale.make_params(cfg, nranks=2, rank=1)
    assert L.sale_workspace_bytes(C.byref(p)) == 0  # NULL id with nranks=2 is invalid


def test_workspace_scales_with_mesh(L):
    c3, _ = configs.config("C3")
    b = sale.workspace_bytes(c3)
    cells = 320 ** 3
    # Lagrange: 12 node + 4 cell arrays + scratch, fp64
    assert 16 * 8 * cells < b < 20 * 8 * cells


def test_null_safety(L):
    L.sale_destroy(None)
    assert L.sale_last_error(None) == b"null context"
    assert L.sale_step(None, 1, None) == sale.EINVAL
