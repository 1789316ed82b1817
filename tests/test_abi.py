"""The C-ABI library loads without a GPU and exports every entry point the header declares."""
import ctypes
import re
from pathlib import Path

from paper_2511_05814_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "moeb200.h").read_text()
    return sorted(set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_native.EXPORTED) == names


def test_abi_version_and_error_channel():
    lib = _native.load_library()
    assert lib.moe_abi_version() == 2
    assert isinstance(lib.moe_last_error(), bytes)


def test_invalid_config_is_rejected_before_any_device_work():
    lib = _native.load_library()
    # K > C must be refused by validation (simulate.py:148-151) without touching CUDA
    st = lib.moe_replay_policy(None, 4, 3, 8, 2, 0, 1.0, 1, None, None, None)
    assert st == _native.MOE_INVALID_CONFIG
    assert b"cannot fit" in lib.moe_last_error()
    st = lib.moe_replay_policy(None, 4, 2, 300, 4, 0, 1.0, 1, None, None, None)
    assert st == _native.MOE_INVALID_CONFIG


def test_engine_struct_layout_matches_header():
    # 8 int32 + double + int64 + float + 4 int32 + (pad) int64 + 2 int32 (moe_engine_config)
    assert ctypes.sizeof(_native.EngineConfigC) == 96
    # 11 int64 + double + 2 int64 (moe_stats)
    assert ctypes.sizeof(_native.StatsC) == 14 * 8
    # 4 double + 5 int64 + double + 2 int64 + double + int64 + double + int64 + 2 double
    assert ctypes.sizeof(_native.KernelTimesC) == 18 * 8
