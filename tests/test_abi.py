"""CPU: the C-ABI library loads and exports every symbol include/fdg.h declares;
host-only entry points (no device work) match the reference."""
import ctypes as C
import subprocess

import numpy as np
import pytest

from paper_2406_13984_b200 import _lib


def test_library_exports_header_symbols():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 50
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and the dynamic symbol table agrees (no C++ mangling at the boundary)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported
    assert set(_lib.SIGNATURES) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    archs = {tok for tok in out.split() if tok.startswith("sm_")}
    assert all("sm_100" in a for a in archs), out


def test_host_batch_seed_and_partition(golden):
    from paper_2406_13984_b200 import featdrive as fd
    for row, want in zip(golden["bs_in"], golden["bs_out"]):
        assert fd.batch_seed(*map(int, row)) == int(want)
    chunks = fd.partition_epoch(np.arange(100, dtype=np.uint64), 7, 99)
    np.testing.assert_array_equal(np.concatenate(chunks), golden["part_small"])
    assert [len(c) for c in chunks] == [7] * 14 + [2]
    flat = np.concatenate(fd.partition_epoch(np.arange(1000, dtype=np.uint64), 20, 0xF7A9D7D3C8F55CC3))
    assert sorted(flat.tolist()) == list(range(1000))


def test_partition_matches_reference_order(golden, port):
    from paper_2406_13984_b200 import featdrive as fd
    order = np.concatenate(fd.partition_epoch(np.arange(1000, dtype=np.uint64), 20, port.hash_combine(0, 0)))
    np.testing.assert_array_equal(order, golden["part_order"])
    with pytest.raises(fd.InvalidArgument):
        fd.partition_epoch(np.arange(3, dtype=np.uint64), 0, 1)


def test_library_sets_hardware_queue_default():
    """Loading libfdg.so sets CUDA_DEVICE_MAX_CONNECTIONS=32 (the runner's 19 streams would share
    the default 8 hardware queues) unless the process already chose a value."""
    code = ("import ctypes, sys; ctypes.CDLL(sys.argv[1]); libc = ctypes.CDLL(None); "
            "libc.getenv.restype = ctypes.c_char_p; print(libc.getenv(b'CUDA_DEVICE_MAX_CONNECTIONS').decode())")
    import os
    import sys
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    out = subprocess.run([sys.executable, "-c", code, _lib.LIB_PATH], capture_output=True, text=True, env=env)
    assert out.stdout.strip() == "32", out.stderr
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "4"
    out = subprocess.run([sys.executable, "-c", code, _lib.LIB_PATH], capture_output=True, text=True, env=env)
    assert out.stdout.strip() == "4", out.stderr
