"""The C++ drop-in (include/featdrive_gpu.hpp): tests/cpp/set_loop.cpp is the reference's
SET loop written against the reference's API. It compiles against the reference headers
(oracle/_ref/set_loop_ref, built here from /root/reference) and against the drop-in with
only the include and the top-level namespace changed; on the GPU both binaries must print
the same per-batch records, the same per-node protocol outcome and the same error behaviour
on a dataset written by the reference generator."""
import os
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2406_13984_b200")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "set_loop_ref")


def _build(tmp_path):
    exe = str(tmp_path / "set_loop")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/set_loop.cpp", f"-L{LIBDIR}", "-lfdg", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                   check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


def test_same_source_builds_against_the_reference():
    """The loop's source is the reference's API: it builds against the reference headers
    (oracle/Makefile target _ref/set_loop_ref) and runs on the CPU."""
    if not os.path.exists(REF_BIN):
        if not os.path.isdir("/root/reference/proj/include"):
            pytest.skip("reference build of set_loop absent and /root/reference not here")
        oracle.build(ref=True)
    assert os.access(REF_BIN, os.X_OK)


@pytest.fixture(scope="module")
def ref_dataset(ref, tmp_path_factory):
    d = str(tmp_path_factory.mktemp("setloop"))
    ref.generate_dataset(d, 5000, 16, 12, 7)
    return d


@pytest.mark.gpu
@pytest.mark.parametrize("slots,batches", [(900, 8), (320, 12), (5000, 6)])
def test_set_loop_equals_reference_loop(tmp_path, ref_dataset, slots, batches):
    """Same source, two builds: the per-batch (nodes, edges, trainer checksum, hits, loads,
    evictions), the per-node protocol batch (alias lists and counters), the mapping entry
    after release and the out_of_range behaviour all equal the reference's."""
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/set_loop_ref not built")
    args = [ref_dataset, str(slots), str(batches)]
    want = subprocess.run([REF_BIN] + args, capture_output=True, text=True, timeout=600)
    got = subprocess.run([_build(tmp_path)] + args, capture_output=True, text=True, timeout=600)
    assert want.returncode == 0, want.stderr
    assert got.returncode == 0, got.stderr
    assert got.stdout.splitlines() == want.stdout.splitlines()
    assert "out_of_range ok" in got.stdout and got.stdout.count("\n") == batches + 3


@pytest.mark.gpu
def test_set_loop_errors_match_reference(tmp_path):
    """A missing dataset fails the same way in both builds (std::system_error from open)."""
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/set_loop_ref not built")
    missing = str(tmp_path / "nope")
    want = subprocess.run([REF_BIN, missing, "100"], capture_output=True, text=True)
    got = subprocess.run([_build(tmp_path), missing, "100"], capture_output=True, text=True)
    assert want.returncode == got.returncode == 1
    assert got.stderr == want.stderr
