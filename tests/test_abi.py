"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and validates arguments on the host (no GPU needed: every
case below fails validation before any device call)."""
import ctypes
import os
import re

import pytest

import paper_2411_05007_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "svdq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svdq_[a-z0-9_]+)\s*\(", src)))


def test_every_header_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 15
    lib = P.abi.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(P.EXPORTS) == syms


def test_binding_names_match_abi():
    for s in header_symbols():
        assert hasattr(P, s), f"binding lacks {s}"


def test_sizes():
    assert P.svdq_act_buffer_sizes("nvfp4", 4608, 3072, 32) == (4608 * 1536, 4608 * 192, 4608 * 64)
    # 129 rows pad to 256 in the 128x4 scale layout
    assert P.svdq_act_buffer_sizes("nvfp4", 129, 128, 0)[1] == 256 * 8
    assert P.svdq_act_buffer_sizes("int4", 129, 128, 16) == (129 * 64, 129 * 2 * 2, 129 * 16 * 2)
    assert P.svdq_weight_buffer_sizes("nvfp4", 3072, 9216, 32) == (9216 * 1536, 9216 * 192, 32 * 3072 * 2,
                                                                   9216 * 32 * 2)


@pytest.mark.parametrize("args,status", [
    (("nvfp4", 0, 64, 16), 2), (("nvfp4", 8, 96, 16), 2), (("nvfp4", 8, 64, 24), 3),
    (("nvfp4", 8, 64, 144), 3), (("int4", 8, 0, 0), 2)])
def test_size_validation(args, status):
    with pytest.raises(P.SvdqError) as e:
        P.svdq_act_buffer_sizes(*args)
    assert e.value.status == status


def test_status_strings_and_last_error():
    assert P.svdq_status_string(0) == "SVDQ_OK"
    assert P.svdq_status_string(3) == "SVDQ_ERR_RANK"
    with pytest.raises(P.SvdqError):
        P.svdq_weight_buffer_sizes("nvfp4", 64, 20, 16)
    assert "N" in P.svdq_last_error()


def test_null_pointer_rejected_before_device():
    lib = P.abi.lib()
    L = P.abi.svdq_linear()
    L.fmt, L.K, L.N, L.rank = 0, 128, 64, 16
    st = lib.svdq_quantize_act_lowrank_down(ctypes.byref(L), None, 0, 8, 128, None, None, None, None)
    assert st == 1
    st = lib.svdq_gemm_w4a4_lowrank_up(None, None, None, None, 8, None, 0, 64, None)
    assert st == 1
    L.rank = 20
    st = lib.svdq_quantize_act_lowrank_down(ctypes.byref(L), None, 0, 8, 128, None, None, None, None)
    assert st == 3


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2411_05007_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f


def test_grouped_argument_validation_before_device():
    """Grouped entry points reject bad group sizes / NULL arrays on the host, before any launch."""
    lib = P.abi.lib()
    st = lib.svdq_gemm_w4a4_lowrank_up_grouped(0, None, None, None, None, None, None, 0, None, None)
    assert st == 1
    st = lib.svdq_gemm_w4a4_lowrank_up_grouped(5, None, None, None, None, None, None, 0, None, None)
    assert st == 1
    st = lib.svdq_gemm_w4a4_lowrank_up_grouped(2, None, None, None, None, None, None, 0, None, None)
    assert st == 1
    st = lib.svdq_quantize_act_lowrank_down_grouped(0, None, None, 0, None, None, None, None, None, None)
    assert st == 1
    st = lib.svdq_quantize_act_lowrank_down_grouped(9, None, None, 0, None, None, None, None, None, None)
    assert st == 1
    # fp16 activations are accepted by the grouped K1 (row-tile kernel); the NULL X is rejected
    L = P.abi.svdq_linear()
    L.fmt, L.K, L.N, L.rank = 0, 128, 64, 16
    arr = (ctypes.POINTER(P.abi.svdq_linear) * 1)(ctypes.pointer(L))
    one = (ctypes.c_void_p * 1)(None)
    i64 = (ctypes.c_int64 * 1)(8)
    st = lib.svdq_quantize_act_lowrank_down_grouped(1, arr, one, 1, i64, i64, one, one, one, None)
    assert st == 1


def test_offline_and_fused_argument_validation_before_device():
    """Layer-boundary fusion, refinement, GPTQ and alpha search reject bad arguments on the host."""
    lib = P.abi.lib()
    # fused next-layer K2: group size, NULL arrays, bad activation
    assert lib.svdq_gemm_w4a4_lowrank_up_fused_next(0, None, None, None, None, None, None, None, 0, None, None, None,
                                                    None, 0, None) == 1
    assert lib.svdq_gemm_w4a4_lowrank_up_fused_next(5, None, None, None, None, None, None, None, 0, None, None, None,
                                                    None, 0, None) == 1
    wsb = ctypes.c_size_t()
    assert lib.svdq_gemm_fused_next_workspace(1, None, None, None, ctypes.byref(wsb)) == 1
    L = P.abi.svdq_linear()
    arr = (ctypes.POINTER(P.abi.svdq_linear) * 1)(ctypes.pointer(L))
    i64 = (ctypes.c_int64 * 1)(8)
    assert lib.svdq_gemm_w4a4_lowrank_up_fused_next(1, arr, None, None, None, i64, None, arr, 7, None, None, None,
                                                    None, 0, None) == 1
    # refinement: negative iteration count, NULL pointers
    best = ctypes.c_int32()
    obj = (ctypes.c_double * 1)()
    assert lib.svdq_refine_lowrank(None, 0, 8, 64, None, None, 64, 64, 16, 0, 0, 1.0, -1, 0, 0.01, None,
                                   ctypes.byref(best), obj, None, 0, None) == 1
    # GPTQ / alpha search workspaces: M_cal < 1
    assert lib.svdq_quantize_residual_gptq_workspace(0, 64, 64, ctypes.byref(wsb)) == 2
    assert lib.svdq_quantize_weights_gptq_workspace(0, 64, 64, 16, ctypes.byref(wsb)) == 2
    assert lib.svdq_search_alpha_workspace(0, 0, 64, 64, 16, ctypes.byref(wsb)) == 2
    assert lib.svdq_refine_lowrank_workspace(0, 0, 64, 64, 16, 0, ctypes.byref(wsb)) == 2
