"""libm4d.so loads on a GPU-less host and exports every symbol include/m4d.h declares."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "m4d.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(m4d_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2101_08878_b200 import native

    lib = native.lib()
    names = declared_symbols()
    assert len(names) > 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert not [n for n in names if n not in native.SIGNATURES]


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2101_08878_b200", "libm4d.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_needed_for_load_and_device_count():
    from paper_2101_08878_b200 import native

    assert native.device_count() >= 0
    assert native.lib().m4d_version() >> 16 == 1


def test_error_codes_map_to_reference_exceptions():
    from paper_2101_08878_b200 import errors, native

    assert isinstance(native.error_for(native.ERR_TRUNCATION, "x"), errors.TruncationError)
    assert isinstance(native.error_for(native.ERR_CANCELLED, "x"), errors.CancelledTransferError)
    assert isinstance(native.error_for(native.ERR_CLOSED, "x"), errors.CommClosedError)
    assert isinstance(native.error_for(native.ERR_CHANNEL, "x"), errors.ChannelError)
    assert isinstance(native.error_for(native.ERR_CUDA, "x"), errors.TransferError)
    assert native.error_for(native.ERR_STARTUP, "x", rank=3).rank == 3


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2101_08878_b200")
    for dirpath, _dirs, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f), encoding="utf-8").read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f


def test_fast_path_extension_binds_to_the_same_library():
    from paper_2101_08878_b200 import native

    fast = native.fast()
    assert fast is native.fast()
    assert fast.progress.__doc__ and fast.post.__doc__
    import pytest

    with pytest.raises(TypeError):
        fast.post(0)
