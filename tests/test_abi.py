"""The C-ABI library loads and exports every symbol include/*.h declares; host-only calls
(no GPU needed) behave as documented.  CPU only."""
import ctypes

import numpy as np
import pytest

from paper_2605_17821_b200 import tc


def test_every_declared_symbol_is_exported():
    names = tc.header_symbols()
    expected = {"tc_status_string", "tc_last_error", "tc_abi_version", "tc_ctx_create", "tc_ctx_destroy",
                "tc_ctx_check", "tc_ctx_launches", "tc_diff_bound", "tc_diff_encode", "tc_stage_host",
                "tc_comm_get_unique_id", "tc_comm_init", "tc_comm_destroy", "tc_replicate_peer",
                "tc_diff_apply", "tc_synth_base", "tc_synth_step", "tc_host_alloc", "tc_host_free", "tc_diff_bound_range", "tc_diff_encode_range"}
    assert expected <= set(names), set(names) ^ expected
    for n in names:
        assert getattr(tc.LIB, n) is not None


def test_status_strings_and_version():
    assert tc.LIB.tc_abi_version() == 1
    assert tc._status_string(0) == "TC_OK"
    assert tc._status_string(5) == "TC_ERR_CORRUPT"
    assert tc._status_string(6) == "TC_ERR_PROTOCOL"
    assert tc._status_string(99) == "TC_ERR_UNKNOWN"


@pytest.mark.parametrize("sizes,wb,T,C", [
    ([0], [4], 4096, 1 << 28), ([6], [4], 4096, 1 << 28), ([3], [2], 4096, 4096),
    ([1000, 2000, 3000], [2, 4, 4], 64, 256), ([70000, 5], [2, 4], 32, 4096),
    ([1557611200, 1557611200, 1557611200, 1557611200], [2, 4, 4, 4], 4096, 1 << 28),
])
def test_bound_matches_oracle_closed_form(tco, sizes, wb, T, C):
    assert tc.diff_bound(sizes, wb, T, C) == tco.worst_case_bytes(sizes, wb, T, C)


def test_bound_rejects_bad_options():
    with pytest.raises(tc.TcError) as e:
        tc.diff_bound([10], [4], tile_words=48)
    assert e.value.status == tc.ERR_INVALID
    with pytest.raises(tc.TcError):
        tc.diff_bound([10], [4], tile_words=64, chunk_words=96)
    with pytest.raises(tc.TcError):
        tc.diff_bound([10], [3])
    with pytest.raises(tc.TcError):
        tc.diff_bound([10] * 17, [4] * 17)


def test_host_side_argument_errors_need_no_gpu():
    # NULL ctx is rejected before anything touches the device
    segs = tc.layout_segments([10], [4])
    ob = ctypes.c_uint64(0)
    rc = tc.LIB.tc_diff_encode(None, segs, 1, None, 1, 0, None, 0, ctypes.byref(ob), None)
    assert rc == tc.ERR_INVALID
    rc = tc.LIB.tc_diff_apply(None, None, None, None, 1, 0, None, None, 1, None)
    assert rc == tc.ERR_INVALID
    rc = tc.LIB.tc_replicate_peer(None, None, None, None, 0, None, 0, None)
    assert rc == tc.ERR_INVALID
    assert "NULL" in tc.LIB.tc_last_error().decode() or tc.LIB.tc_last_error()


def test_ctx_create_without_gpu_reports_cuda_error():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = tc.LIB.tc_ctx_create(0, ctypes.byref(h))
    assert rc == tc.ERR_CUDA and not h.value


def test_bound_range_sums_to_bound(tco):
    n, w, T, C = 100003, 4, 256, 4096
    full = tc.diff_bound([n], [w], T, C)
    nch = -(-n // C)
    parts = [tc.diff_bound_range(n, w, c, 3, T, C) for c in range(0, nch, 3)]
    assert sum(parts) == full
    with pytest.raises(tc.TcError):
        tc.diff_bound_range(n, w, nch, 1, T, C)
