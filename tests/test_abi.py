"""The C-ABI library loads and exports every symbol include/primkit/primkit.h
declares; section 1 is the reference ABI (31 functions, same names), and the
struct layouts match the reference header. No compute calls (CPU suite)."""
import ctypes as C
import os

from paper_1910_00078_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "primkit", "primkit.h")

# the reference ABI (/root/reference/proj/include/primkit/primkit.h:114-217)
REFERENCE_SYMBOLS = [
    "primkit_last_error", "primkit_handle_create", "primkit_handle_destroy",
    "primkit_handle_use_fake_clock", "primkit_handle_now_ms", "primkit_handle_set_cache_dir",
    "primkit_handle_counters", "primkit_handle_reset_counters", "primkit_handle_set_seed",
    "primkit_problem_key", "primkit_conv_output_dims", "primkit_solver_count",
    "primkit_solver_name", "primkit_solver_is_applicable", "primkit_solver_is_tunable",
    "primkit_solver_workspace_bytes", "primkit_find_convolution", "primkit_conv_run",
    "primkit_tune", "primkit_perfdb_save", "primkit_perfdb_load", "primkit_fusion_plan_create",
    "primkit_fusion_plan_destroy", "primkit_fusion_add_conv", "primkit_fusion_add_bias",
    "primkit_fusion_add_batchnorm", "primkit_fusion_add_activation", "primkit_fusion_compile",
    "primkit_fusion_output_dims", "primkit_fusion_set_args", "primkit_fusion_execute",
]


def test_header_declares_reference_abi():
    declared = abi.header_symbols(HEADER)
    assert len(REFERENCE_SYMBOLS) == 31
    for s in REFERENCE_SYMBOLS:
        assert s in declared, s
    assert set(abi.SECTION1) == set(REFERENCE_SYMBOLS)
    assert set(declared) == set(abi.SECTION1) | set(abi.SECTION2)


def test_library_exports_every_declared_symbol(lib):
    raw = C.CDLL(lib.path)
    for s in abi.header_symbols(HEADER):
        assert hasattr(raw, s), f"missing export {s}"


def test_internal_symbols_hidden(lib):
    raw = C.CDLL(lib.path)
    # kernel launchers are an internal boundary, not part of the ABI
    assert not hasattr(raw, "pk_cuda_direct_fwd")


def test_struct_layouts():
    # 14 x int64 + 3 enums (ref primkit.h:88-98), padded to 8
    assert C.sizeof(abi.ConvProblem) == 14 * 8 + 3 * 4 + 4
    assert C.sizeof(abi.AlgoPerf) == 64 + 4 + 4 + 8 + 8
    assert C.sizeof(abi.Counters) == 24
    assert abi.AlgoPerf.time_ms.offset == 72


def test_reference_header_layouts_match():
    ref_header = "/root/reference/proj/include/primkit/primkit.h"
    if not os.path.exists(ref_header):
        import pytest
        pytest.skip("reference sources not present")
    ref_syms = abi.header_symbols(ref_header)
    assert sorted(ref_syms) == sorted(REFERENCE_SYMBOLS)
    text = open(ref_header).read()
    for enum_line in ("PRIMKIT_STATUS_INTERNAL = 20", "PRIMKIT_ALGO_IMPLICIT_GEMM = 4",
                      "PRIMKIT_BN_SPATIAL = 1", "PRIMKIT_ACT_TANH = 3", "PRIMKIT_BF16 = 1"):
        assert enum_line in text
        assert enum_line in open(HEADER).read()


def test_channel_pitch(lib):
    assert [lib.channel_pitch(c) for c in (1, 3, 8, 9, 64, 65)] == [8, 8, 8, 16, 64, 72]
