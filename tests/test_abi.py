"""The C-ABI library loads without a GPU, exports every function include/bbc.h declares,
and carries sm_100a code (CPU only; no compute calls)."""

import ctypes
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions() -> list[str]:
    text = (ROOT / "include" / "bbc.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bbc_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_documented_entry_points():
    names = declared_functions()
    for required in ("bbc_graph_create", "bbc_graph_create_device", "bbc_count", "bbc_graph_destroy",
                     "bbc_last_error", "bbc_block_work", "bbc_task_order"):
        assert required in names


def test_library_exports_every_declared_symbol(native_built):
    from paper_2601_17707_b200 import _lib

    L = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(_lib.EXPORTED_SYMBOLS) <= set(declared_functions())


def test_library_has_sm100a_code(native_built):
    from paper_2601_17707_b200 import _lib

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "bbc.h"\nint main(void){ bbc_opts o = {0}; (void)o; return 0; }\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-c", str(src), "-o",
                        str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_gpu_means_loud_failure(native_built):
    from conftest import has_gpu
    from paper_2601_17707_b200 import DeviceError, _lib

    if has_gpu():
        pytest.skip("a GPU is visible")
    assert _lib.device_count() == 0
    with pytest.raises((DeviceError, ValueError)):
        _lib.DeviceGraph.from_host(2, 2, [0], [0], [1])
