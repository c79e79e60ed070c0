"""CPU-side checks of the C-ABI boundary: libcadet.so builds, loads, and exports every symbol
include/cadet.h declares; the binding's names match.  No compute calls (no GPU here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cadet.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_\s\*]*?\b(cadet_[a-z0-9_]+)\s*\(", src,
                                 flags=re.M)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("cadet_mask_plan", "cadet_attn_core_forward", "cadet_attn_core_backward", "cadet_attn_forward",
              "cadet_attn_backward", "cadet_heads_forward", "cadet_heads_loss_backward", "cadet_chunk",
              "cadet_pack", "cadet_poll"):
        assert f in fns


def test_library_builds_loads_and_exports_all_symbols():
    from paper_2602_11410_b200 import build, _lib
    build.build()
    import ctypes
    L = ctypes.CDLL(build.LIB)
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, f"declared in cadet.h but not exported: {missing}"
    assert set(header_functions()) == set(_lib.SIGNATURES), "binding names must equal the header's"
    assert _lib.lib().cadet_abi_version() == 1


def test_default_config_matches_paper_constants():
    from paper_2602_11410_b200 import _lib
    c = _lib.default_config(352, 4)
    assert c.head_dim == 88 and c.delta_delay_ms == 3_600_000
    assert c.rope_delta_t_max_ms == 31_536_000_000 and c.rope_phi_min == 1e-4 and c.rope_base == 600000.0
    assert c.mask_flags == _lib.CADET_MASK_TIME


def test_host_validation_errors_without_gpu():
    """Host-detected errors return synchronously (no device work is enqueued)."""
    import ctypes as C
    from paper_2602_11410_b200 import _lib
    L = _lib.lib()
    c = _lib.default_config(100, 3)   # d % H != 0
    b = _lib.BatchStruct()
    assert L.cadet_mask_plan(C.byref(c), C.byref(b), None, 0, None) == 1
    c = _lib.default_config(64, 1)    # head_dim 64 ok, unknown dtype
    c.dtype = 7
    assert L.cadet_mask_plan(C.byref(c), C.byref(b), None, 0, None) == 1
    c = _lib.default_config(2048, 256)  # head_dim 8 is not a supported head size; H > 128
    assert L.cadet_mask_plan(C.byref(c), C.byref(b), None, 0, None) == 1
    c = _lib.default_config(8192, 256)  # head_dim 32 ok, but H > 128
    assert L.cadet_mask_plan(C.byref(c), C.byref(b), None, 0, None) == 1
    c = _lib.default_config(64, 1)    # the fp32 parity mode: sizes follow the fp32 layout
    c.dtype = 1
    c16 = _lib.default_config(64, 1)
    assert L.cadet_attn_saved_bytes(C.byref(c), 1000) > L.cadet_attn_saved_bytes(C.byref(c16), 1000)
    assert L.cadet_attn_bwd_ds_bytes(C.byref(c), 1, 1000, 1000) == 0
    assert L.cadet_gemm_fp32_workspace_bytes(100, 64, 30) == 2 * 12800 + 2 * 8192  # K padded to 32
    g = C.c_void_p(256)  # never dereferenced: boundaries are validated on the host first
    assert L.cadet_bucketize(g, 4, (C.c_int32 * 2)(4, 4), 2, g, g, None) == 1   # not strictly increasing
    assert L.cadet_bucketize(g, 4, (C.c_int32 * 1)(4), 0, g, g, None) == 1      # nb < 1
    c = _lib.default_config(64, 1)    # deterministic mode is bf16-only
    c.dtype, c.deterministic = 1, 1
    assert L.cadet_mask_plan(C.byref(c), C.byref(b), None, 0, None) == 9
    assert L.cadet_gemm(0, 32, 32, None, 0, None, 0, None, 1, None, None) == 1


def test_next_rows_host_validation_and_size_queries_without_gpu():
    """NEXT-3 / NEXT-4 / two-pass backward entry points: argument errors are host-detected and
    returned synchronously (no CUDA call), and the size queries follow their documented formulas."""
    import ctypes as C
    from paper_2602_11410_b200 import _lib
    L = _lib.lib()
    E_ARG = 1
    # RMSNorm: d % 8 == 0 and d <= 1024
    g = C.c_void_p(256)  # never dereferenced: the call fails before any device work
    assert L.cadet_rmsnorm_forward(g, g, 4, 1025, g, g, None) == E_ARG
    assert L.cadet_rmsnorm_forward(g, g, 4, 12, g, g, None) == E_ARG
    assert L.cadet_rmsnorm_backward(g, None, g, g, None, 4, 64, g, g, None) == E_ARG   # gamma null
    # FFN: d % 32 == 0, weights non-null
    assert L.cadet_ffn_forward(g, g, g, None, 4, 48, 4, g, g, g, None) == E_ARG
    assert L.cadet_ffn_forward(g, None, g, None, 4, 64, 4, g, g, g, None) == E_ARG
    assert L.cadet_ffn_workspace_bytes(1000, 256, 4) == -(-1000 * 256 * 4 * 2 // 256) * 256
    # AdamW: step >= 1 and 16-byte-aligned fp32 buffers
    cfg = _lib.AdamWConfig()
    L.cadet_default_adamw_config(C.byref(cfg))
    assert abs(cfg.lr - 1e-4) < 1e-9 and abs(cfg.beta2 - 0.999) < 1e-7 and cfg.weight_decay == 0.0
    assert L.cadet_adamw_step(C.byref(cfg), 0, g, g, g, g, None, 16, None) == E_ARG
    assert L.cadet_adamw_step(C.byref(cfg), 1, C.c_void_p(260), g, g, g, None, 16, None) == E_ARG
    assert L.cadet_bf16_to_f32(C.c_void_p(264), g, 8, None) == E_ARG
    # two-pass backward region: dS^T slots bounded like the plan's visit lists, times H x 32 KB
    c = _lib.default_config(1024, 8)
    n, T, L_max = 136, 65536, 2048
    nq, hm = (T + 127) // 128 + n, (L_max + 127) // 128 + 3
    slots = nq * (hm + 1) // 2 + hm
    assert L.cadet_attn_bwd_ds_bytes(C.byref(c), n, T, L_max) == -(-slots * 8 * 128 * 128 * 2 // 256) * 256
    assert L.cadet_attn_bwd_ds_bytes(C.byref(c), n, T, 1 << 30) == 0   # bound overflows: no region
