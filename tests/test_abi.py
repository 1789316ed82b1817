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
    assert lib.moe_abi_version() == 4
    assert isinstance(lib.moe_last_error(), bytes)


def test_invalid_config_is_rejected_before_any_device_work():
    lib = _native.load_library()
    # K > C must be refused by validation (simulate.py:148-151) without touching CUDA
    st = lib.moe_replay_policy(None, 4, 3, 8, 2, 0, 1.0, 1, None, None, None)
    assert st == _native.MOE_INVALID_CONFIG
    assert b"cannot fit" in lib.moe_last_error()
    st = lib.moe_replay_policy(None, 4, 2, 300, 4, 0, 1.0, 1, None, None, None)
    assert st == _native.MOE_INVALID_CONFIG


def test_engine_struct_layout_matches_header(tmp_path):
    """Every ctypes mirror has the C header's size and field offsets (compiled with gcc)."""
    import subprocess

    structs = {"moe_engine_config": _native.EngineConfigC, "moe_stats": _native.StatsC,
               "moe_kernel_times": _native.KernelTimesC}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT / "include" / "moeb200.h"}"',
             "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], check=True, capture_output=True,
                                                         text=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, f"{cname}.{f}"
