"""CPU tests of the host side: the Python mirror of the reference API, the
C-ABI library (loads, exports every declared symbol, validates like the
reference before touching any device), and the schema table."""
import math
import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2504_13821_b200 as rc
from paper_2504_13821_b200 import (
    AliasError,
    Backend,
    BoundsError,
    ConfigError,
    MatrixBuffer,
    MatrixView,
    OpKind,
    ShapeError,
    Side,
    SplitError,
    Threshold,
    TileLimitError,
    Trans,
    TriangularSpec,
    Uplo,
    _lib,
)

HEADER = Path(__file__).resolve().parents[1] / "include" / "rectri_cu.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(rectri_cu_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert lib.rectri_cu_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_flags_and_variant_strings():
    # flags.cpp:5-40
    assert rc.parse_side("left") == Side.Left and rc.parse_uplo("upper") == Uplo.Upper
    assert rc.parse_trans("c") == Trans.ConjTrans and rc.parse_diag("unit") == rc.Diag.Unit
    with pytest.raises(ConfigError):
        rc.parse_side("middle")
    assert rc.variant_string(TriangularSpec()) == "left-lower-n-nonunit"
    assert rc.variant_string(TriangularSpec(Side.Right, Uplo.Upper, Trans.Trans, rc.Diag.Unit)) == \
        "right-upper-t-unit"
    assert rc.effective_op(Trans.ConjTrans) == Trans.Trans
    with pytest.raises(ConfigError):
        rc.validate(TriangularSpec(alpha=math.nan))
    # 16 distinct variants (test_variants.cpp:37-45)
    seen = {rc.variant_string(TriangularSpec(Side(s), Uplo(u), Trans(t), rc.Diag(d)))
            for s in (0, 1) for u in (0, 1) for t in (0, 1) for d in (0, 1)}
    assert len(seen) == 16


def test_matrix_views():
    # matrix.hpp / test_matrix.cpp:9-75
    assert rc.split_half(5) == 2 and rc.split_half(2) == 1
    with pytest.raises(SplitError):
        rc.split_half(1)
    buf = MatrixBuffer(6, 5, torch.float64, "cpu")
    v = buf.view()
    s = v.subview(1, 2, 3, 2)
    assert (s.rows(), s.cols(), s.row_offset(), s.col_offset(), s.leading_dim()) == (3, 2, 1, 2, 6)
    with pytest.raises(BoundsError):
        v.subview(4, 0, 3, 1)
    s.tensor()[:] = 7.0
    t = buf.tensor()
    assert t[1:4, 2:4].eq(7).all() and t.sum().item() == 7.0 * 6
    assert rc.overlaps(v.subview(0, 0, 3, 3), v.subview(2, 2, 2, 2))
    assert not rc.overlaps(v.subview(0, 0, 3, 3), v.subview(3, 0, 3, 3))
    assert not rc.overlaps(v.subview(0, 0, 0, 3), v)
    other = MatrixBuffer(6, 5, torch.float64, "cpu")
    assert not rc.overlaps(v, other.view())


def _cpu(a):
    return MatrixBuffer.from_tensor(torch.as_tensor(np.asarray(a, dtype=np.float64)), device="cpu")


def test_validation_order_before_any_device_work():
    """check_problem (recursion.cpp:50-67): Config, Shape, Alias -- raised by
    the C-ABI before it looks at memory, so testable on CPU."""
    spec = TriangularSpec()
    a = _cpu(np.eye(4))
    b = _cpu(np.ones((4, 2)))
    with pytest.raises(ConfigError):
        rc.rec_trsm(spec, a.cview(), b.view(), Threshold(0))
    with pytest.raises(ConfigError):
        rc.rec_trsm(TriangularSpec(alpha=math.inf), a.cview(), b.view())
    with pytest.raises(ConfigError):
        rc.rec_trmm(spec, a.cview(), b.view(), Threshold(2), Backend(parallel_width=0))
    with pytest.raises(ShapeError):
        rc.rec_trmm(spec, _cpu(np.ones((4, 3))).cview(), b.view(), Threshold(2))
    with pytest.raises(ShapeError):
        rc.rec_trsm(spec, a.cview(), _cpu(np.ones((5, 2))).view(), Threshold(2))
    with pytest.raises(ShapeError):  # Right side wants B.cols == n
        rc.rec_trsm(TriangularSpec(Side.Right), a.cview(), b.view(), Threshold(2))
    shared = MatrixBuffer(8, 8, torch.float64, "cpu", 1.0)
    v = shared.view()
    with pytest.raises(AliasError):
        rc.rec_trmm(spec, v.subview(0, 0, 4, 4).as_const(), v.subview(3, 3, 4, 4), Threshold(2))
    # Config is checked before Shape (threshold 0 with a bad shape).
    with pytest.raises(ConfigError):
        rc.rec_trsm(spec, _cpu(np.ones((4, 3))).cview(), b.view(), Threshold(0))
    # Degenerate shapes are no-ops (recursion.cpp:170, 183) -- no device needed.
    rc.rec_trsm(spec, a.cview(), MatrixBuffer(4, 0, torch.float64, "cpu").view(), Threshold(2))
    rc.rec_trmm(spec, MatrixBuffer(0, 0, torch.float64, "cpu").cview(),
                MatrixBuffer(0, 2, torch.float64, "cpu").view())
    # Base kernel: tile limit (base_kernels.cpp:16-33).
    big = _cpu(np.eye(300))
    with pytest.raises(TileLimitError):
        rc.trsm_base(spec, big.cview(), _cpu(np.ones((300, 1))).view())
    with pytest.raises(AliasError):
        rc.trsm_base(spec, v.subview(0, 0, 4, 4).as_const(), v.subview(2, 2, 4, 4))
    # gemm shape / alias (gemm.cpp:164-176)
    with pytest.raises(ShapeError):
        rc.gemm(1.0, Trans.NoTrans, _cpu(np.ones((3, 2))).cview(), Trans.NoTrans, _cpu(np.ones((3, 4))).cview(),
                0.0, _cpu(np.ones((3, 4))).view())
    with pytest.raises(AliasError):
        rc.gemm(1.0, Trans.NoTrans, v.subview(0, 0, 2, 2).as_const(), Trans.NoTrans,
                v.subview(4, 4, 2, 2).as_const(), 0.0, v.subview(1, 1, 2, 2))


def test_schema_table_cpu(golden):
    # recursion.cpp:18-46 evaluated by the library vs the reference's table.
    for row in golden["schema"]:
        op, side, uplo, trans = (int(x) for x in row[:4])
        sc = rc.schema_for(OpKind(op), TriangularSpec(Side(side), Uplo(uplo), Trans(trans)))
        got = [sc.first_block == 1, int(sc.update.off_trans), sc.update.off_on_left, int(sc.update.read_half),
               int(sc.update.write_half), sc.update.sign, sc.update.carries_alpha, sc.second_block == 1]
        assert [float(x) for x in got] == [float(x) for x in row[4:]], row


def test_schema_examples():
    # test_recursion.cpp:60-91
    lln = TriangularSpec()
    trsm = rc.schema_for(OpKind.Trsm, lln)
    assert trsm.first_block == rc.DiagBlock.A11 and trsm.second_block == rc.DiagBlock.A22
    assert trsm.update.read_half == rc.BHalf.B1 and trsm.update.write_half == rc.BHalf.B2
    assert trsm.update.sign == -1.0 and not trsm.update.carries_alpha
    llt = TriangularSpec(trans=Trans.Trans)
    t = rc.schema_for(OpKind.Trmm, llt)
    assert t.first_block == rc.DiagBlock.A11 and t.update.read_half == rc.BHalf.B2 and t.update.carries_alpha
    n = rc.schema_for(OpKind.Trmm, lln)
    assert n.first_block == rc.DiagBlock.A22 and n.update.write_half == rc.BHalf.B2
    assert rc.schema_for(OpKind.Trmm, TriangularSpec(trans=Trans.ConjTrans)).first_block == rc.DiagBlock.A11


def test_errors_map_one_to_one():
    from paper_2504_13821_b200.errors import raise_for_status

    for code, cls in ((1, ConfigError), (2, ShapeError), (3, AliasError), (5, TileLimitError),
                      (7, BoundsError), (8, SplitError), (6, rc.CudaError)):
        with pytest.raises(cls):
            raise_for_status(code, "x")
    with pytest.raises(rc.SingularityError) as e:
        raise_for_status(4, "", 17)
    assert e.value.index() == 17
    raise_for_status(0, "")


def test_cpp_dropin_compiles_against_reference_style_headers():
    """Reference-style user code (#include "rectri/recursion.hpp",
    rec_trsm<float>(spec, a.view(), b.view(), Threshold{..}, Backend::par()))
    compiles against the drop-in headers and links to librectri_cu.so."""
    from paper_2504_13821_b200 import build as b

    exe = b.build_dropin_example()
    assert exe.exists()
