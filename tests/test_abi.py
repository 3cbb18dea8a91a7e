"""CPU-only checks of the C-ABI boundary (no kernel launches): the library loads, exports every
symbol include/fhwt.h declares, and validates arguments with the documented status codes."""
import ctypes
import os
import re

import pytest

import paper_1002_2184_b200 as fhwt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "fhwt.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fhwt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = fhwt.lib()
    names = _declared_symbols()
    assert len(names) >= 20, names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", fhwt.lib_path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_filter_bank_is_section_ii_set():
    fb = fhwt.haar_filter_bank()
    s = 1.0 / 2.0 ** 0.5
    assert list(fb.b0) == pytest.approx([s, s], rel=1e-15)
    assert list(fb.b1) == pytest.approx([-s, s], rel=1e-15)
    assert list(fb.a0) == pytest.approx([s, s], rel=1e-15)
    assert list(fb.a1) == pytest.approx([s, -s], rel=1e-15)
    assert fb.M == 2


@pytest.mark.parametrize("args,exc", [
    ((0, 4, 1), fhwt.EmptySignal),
    ((8, 0, 1), fhwt.EmptySignal),
    ((-8, 1, 1), fhwt.InvalidArgument),
    ((7, 1, 1), fhwt.OddLength),
    ((8, 1, 0), fhwt.InvalidLevels),
    ((12, 1, 3), fhwt.InsufficientLength),
])
def test_plan_1d_validation(args, exc):
    with pytest.raises(exc):
        fhwt.Plan1d(*args)


@pytest.mark.parametrize("args,exc", [
    ((0, 8, 1, 1), fhwt.EmptySignal),
    ((8, 8, 0, 1), fhwt.EmptySignal),
    ((3, 8, 1, 1), fhwt.OddLength),
    ((8, 5, 1, 1), fhwt.OddLength),
    ((8, 8, 1, 0), fhwt.InvalidLevels),
    ((8, 12, 1, 3), fhwt.InsufficientLength),
    ((1 << 30, 8, 1, 1), fhwt.InvalidArgument),      # beyond the TMA coordinate range
])
def test_plan_2d_validation(args, exc):
    with pytest.raises(exc):
        fhwt.Plan2d(*args)


def test_unsupported_filter_bank():
    fb = fhwt.haar_filter_bank()
    fhwt.Plan1d(16, 1, 2, fb)                       # the §II set itself is accepted
    fb.b1[0], fb.b1[1] = fb.b1[1], fb.b1[0]          # the Eq. (9) sign convention is a different bank
    with pytest.raises(fhwt.UnsupportedFilter):
        fhwt.Plan1d(16, 1, 2, fb)
    fb = fhwt.haar_filter_bank()
    fb.M = 3
    with pytest.raises(fhwt.UnsupportedFilter):
        fhwt.Plan2d(16, 16, 1, 2, fb)
    fb = fhwt.haar_filter_bank()
    fb.a0[0] *= 2                                    # Eq. (14)'s factor 2 is reading R3's rejected gain
    with pytest.raises(fhwt.UnsupportedFilter):
        fhwt.Plan2d(16, 16, 1, 2, fb)


def test_workspace_sizes():
    # 2-D plans hold 256 B of tile counters (dynamic tile order) after the pass hand-offs
    assert fhwt.Plan2d(2048, 2048, 256, 5).workspace_bytes == 256        # c4: one fused pass
    assert fhwt.Plan2d(32768, 32768, 1, 8).workspace_bytes == 1024 * 1024 * 8 + 256   # c5: fp64 LL_5 hand-off
    assert fhwt.Plan1d(65536, 4096, 10).workspace_bytes == 0             # c2: one pass
    assert 3 * 16 * 8 <= fhwt.Plan1d(1 << 14, 3, 14).workspace_bytes < 3 * 16 * 8 + 256   # fp64 a_10 hand-off


def test_band_offsets_match_mallat_layout():
    assert fhwt.band_offset_1d(1024, 1, 1) == (512, 512)
    assert fhwt.band_offset_1d(1024, 10, 0) == (0, 1)
    assert fhwt.band_offset_2d(512, 512, 1, 1) == (256, 256, 256)            # HL: top-right
    assert fhwt.band_offset_2d(512, 512, 1, 2) == (256 * 512, 256, 256)      # LH: bottom-left
    assert fhwt.band_offset_2d(512, 512, 3, 3) == (64 * 512 + 64, 64, 64)    # HH_3
    with pytest.raises(fhwt.InvalidArgument):
        fhwt.band_offset_2d(512, 512, 1, 4)


def test_null_and_cpu_pointer_rejection():
    L = fhwt.lib()
    st = L.fhwt_analyze_1d(None, None, 8, 1, 1, None)
    assert st == fhwt.InvalidArgument.status
    assert b"null" in L.fhwt_last_error_message()
    import torch
    with pytest.raises(fhwt.InvalidArgument):
        fhwt.analyze_2d(torch.zeros(8, 8), 1)     # no CPU fallback: fails loudly
    assert L.fhwt_plan_destroy(None) == 0
    assert L.fhwt_status_string(8) == b"FHWT_ERR_MISALIGNED"
    assert ctypes.sizeof(fhwt.FilterBank) >= 8 * 8 + 4


@pytest.mark.parametrize("shape,levels", [((8,), 1), ((64,), 3), ((1024,), 10), ((16, 16), 1), ((32, 64), 3),
                                          ((64, 64), 5)])
def test_op_counts_match_the_oracles_instrumented_count(shape, levels):
    """The C-ABI op-count formulas equal the operations the fp64 oracle actually performs (its
    OpCounter counts every sample multiply/add of the direct and fast structures)."""
    import numpy as np

    import oracle as o
    x = np.ones(shape)
    for structure, mode in (("direct", "direct"), ("fast", "fast")):
        ops = o.OpCounter()
        if len(shape) == 1:
            c = o.decompose_1d(x, levels, mode, ops)
        else:
            c = o.analyze_2d(x, levels, mode, ops)
        assert fhwt.op_counts(shape, levels, structure) == (ops.mul, ops.add), (structure, "analysis")
        ops = o.OpCounter()
        if len(shape) == 1:
            o.reconstruct_1d(c, levels, mode, ops)
        else:
            o.synthesize_2d(c, levels, mode, ops)
        assert fhwt.op_counts(shape, levels, structure, synthesis=True) == (ops.mul, ops.add), (structure, "synthesis")
    dm, da = fhwt.op_counts(shape, levels, "direct")
    fm, fa = fhwt.op_counts(shape, levels, "fast")
    assert 4 * fm == dm and 3 * (fm + fa) == dm + da      # PAPER.md:124 "less than quarter"; 1/3 total
    km, ka = fhwt.op_counts(shape, levels, "kernel")
    assert km <= fm and km + ka <= fm + fa
    assert fhwt.op_counts(shape, levels, "fast", batch=7) == (7 * fm, 7 * fa)


def test_huge_batches_are_accepted():
    """batch * h beyond the int32 TMA row range is split into sub-batches, not rejected."""
    p = fhwt.Plan2d(1 << 20, 8, 4096, 1)
    assert p.batch == 4096


def test_plan_pack_ll_rejects_bad_plans():
    L = fhwt.lib()
    assert L.fhwt_plan_pack_ll_2d(None, None, None, None) == 1          # INVALID_ARG: NULL plan
    p1 = fhwt.Plan1d(64, 2, 3)
    assert L.fhwt_plan_pack_ll_2d(p1._h, None, None, None) == 1         # INVALID_ARG: 1-D plan
    p2 = fhwt.Plan2d(64, 64, 1, 3)
    assert L.fhwt_plan_pack_ll_2d(p2._h, None, None, None) == 1         # INVALID_ARG: NULL buffers
    assert L.fhwt_workspace_bytes(p2._h) == L.fhwt_plan_workspace_bytes(p2._h) == 256
