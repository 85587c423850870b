"""The C-ABI library loads on a CPU-only host and exports every symbol the header declares."""

import ctypes
import os
import re

from paper_2408_10731_b200 import _lib

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "trajopt_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(tro_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    assert set(names) == set(_lib.EXPORTS), names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_struct_layouts_match_header():
    # 10 int32 dims; 11 const pointers; 4 doubles + 4 int32; 18 pointers
    assert ctypes.sizeof(_lib.Alg1Dims) == 40
    assert ctypes.sizeof(_lib.Alg1Consts) == 13 * 8
    assert ctypes.sizeof(_lib.Alg1Params) == 4 * 8 + 4 * 4
    assert ctypes.sizeof(_lib.Alg1State) == 23 * 8


def test_host_only_calls():
    lib = _lib.load()
    assert lib.tro_version() >= 1
    assert lib.tro_error_string(0) == b"success"
    assert b"invalid" in lib.tro_error_string(-1)
    assert lib.tro_topk_workspace_bytes(1000, 10) == 8000
    # argument validation happens before any CUDA call
    assert lib.tro_topk_stable_f64(None, 10, 20, None, None, 0, None) == _lib.TRO_EINVAL
    assert lib.tro_kkt_apply_f64(None, 4, None, 1, None, None) == _lib.TRO_EINVAL
    assert lib.tro_alg1_iterate(0, None, None, None, None, None) == _lib.TRO_EINVAL


def test_struct_sizes_match_c_compiler(tmp_path):
    """sizeof / offsetof of every C-ABI struct from gcc equals the ctypes mirror."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        import pytest

        pytest.skip("gcc not available")
    pairs = {
        "tro_alg1_dims": _lib.Alg1Dims, "tro_alg1_consts": _lib.Alg1Consts, "tro_alg1_params": _lib.Alg1Params,
        "tro_alg1_state": _lib.Alg1State, "tro_priest_dims": _lib.PriestDims, "tro_priest_consts": _lib.PriestConsts,
        "tro_priest_io": _lib.PriestIO, "tro_ma_dims": _lib.MaDims, "tro_ma_consts": _lib.MaConsts,
        "tro_ma_state": _lib.MaState, "tro_ma_params": _lib.MaParams, "tro_b2_dims": _lib.B2Dims,
        "tro_b2_consts": _lib.B2Consts, "tro_b2_state": _lib.B2State, "tro_b2_params": _lib.B2Params,
        "tro_val_dims": _lib.ValDims, "tro_val_consts": _lib.ValConsts, "tro_val_io": _lib.ValIO,
        "tro_track_dims": _lib.TrackDims, "tro_mpc_dims": _lib.MpcDims, "tro_mpc_consts": _lib.MpcConsts,
        "tro_mpc_io": _lib.MpcIO,
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{os.path.abspath(HEADER)}"', "int main(void) {"]
    for cname, ct in pairs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in ct._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "sizes.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for cname, ct in pairs.items():
        assert int(got[cname]) == ctypes.sizeof(ct), cname
        for fname, _ in ct._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(ct, fname).offset, f"{cname}.{fname}"
