"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/lasp.h declares,
and its synchronous validation/planning logic behaves as documented (no GPU compute is called)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2404_02882_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    names = N.header_functions()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert set(names) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in ln for ln in out.splitlines() if ".cubin" in ln)


def _shape(B=1, C=1024, H=4, D=64, dt=N.LASP_BF16):
    return N.shape(B, C, H, D, dt)


def test_sizes_and_plan():
    lib = N.lib()
    s = _shape(1, 32768, 16, 64)
    L = lib.lasp_segment_len(ctypes.byref(s))
    assert L % 128 == 0 and L > 0
    nseg = -(-32768 // L)
    assert lib.lasp_cache_bytes(ctypes.byref(s)) == 1 * 16 * nseg * 64 * 64 * 4 + 256  # + the tag
    assert lib.lasp_workspace_bytes(ctypes.byref(s)) >= 16 * nseg * 64 * 64 * 4 + 3 * 16 * 64 * 64 * 4
    # empty rank: one segment slot holds KV_in
    s0 = _shape(2, 0, 3, 32)
    assert lib.lasp_cache_bytes(ctypes.byref(s0)) == 2 * 3 * 32 * 32 * 4 + 256
    # unsupported head_dim -> 0 bytes
    assert lib.lasp_cache_bytes(ctypes.byref(_shape(D=96))) == 0


def _call_fwd(s, lam, ptr=16):
    lib = N.lib()
    lamarr = np.asarray(lam, dtype=np.float32)
    p = ctypes.c_void_p(ptr)
    return lib.lasp_fwd_local(ctypes.byref(s), p, p, p, lamarr.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                              None, p, None, p, p, None)


@pytest.mark.parametrize("lam,status", [([1.5, 0.9, 0.9, 0.9], 2), ([0.0, 0.9, 0.9, 0.9], 2),
                                        ([float("nan"), 0.9, 0.9, 0.9], 2)])
def test_domain_errors(lam, status):
    assert _call_fwd(_shape(), lam) == status
    assert "outside (0, 1]" in N.lib().lasp_last_error().decode()


def test_shape_errors():
    lib = N.lib()
    assert _call_fwd(_shape(D=96), [0.9] * 4) == 7          # UNSUPPORTED
    assert _call_fwd(_shape(B=0), [0.9] * 4) == 1           # SHAPE
    assert _call_fwd(_shape(), [0.9] * 4, ptr=18) == 1      # misaligned pointers
    assert lib.lasp_fwd_local(None, None, None, None, None, None, None, None, None, None, None) == 1


def test_cache_holds_tag_after_states():
    """The cache is the fp32 segment states [B][H][nseg][D][D] (256-byte aligned) plus a 256-byte tag that the
    forward writes and the backward checks on the device (include/lasp.h)."""
    lib = N.lib()
    for B, C, H, D in ((1, 1000, 4, 64), (2, 32768, 16, 128), (1, 0, 3, 32)):
        s = N.shape(B, C, H, D, N.LASP_BF16)
        nseg = max(1, -(-C // lib.lasp_segment_len(ctypes.byref(s))))
        states = B * H * nseg * D * D * 4
        assert lib.lasp_cache_bytes(ctypes.byref(s)) == -(-states // 256) * 256 + 256


def test_workspace_status_rejects_null():
    lib = N.lib()
    assert lib.lasp_workspace_status(None, None) == 1
    assert lib.lasp_workspace_status(ctypes.c_void_p(18), None) == 1


def test_ctx_rejects_bad_rank():
    lib = N.lib()
    out = ctypes.c_void_p()
    assert lib.lasp_ctx_create(3, 2, b"\0" * 128, 0, ctypes.byref(out)) == 3


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(N, "_lib", None)
    with pytest.raises(ImportError):
        N.lib()
