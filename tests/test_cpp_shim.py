"""The C++ drop-in (include/featdrive_gpu.hpp) driven by a reference-shaped SET loop
(tests/cpp/set_loop.cpp): compiles on CPU; on the GPU its per-batch output must
equal the oracle running the same loop."""
import os
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2406_13984_b200")


def _build(tmp_path):
    exe = str(tmp_path / "set_loop")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/set_loop.cpp", f"-L{LIBDIR}", "-lfdg", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                   check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_shim_set_loop_matches_oracle(tmp_path, port):
    from paper_2406_13984_b200 import featdrive as fd
    n, dim, avg, slots = 5000, 16, 12, 900
    out = subprocess.run([_build(tmp_path), str(n), str(dim), str(avg), str(slots)], capture_output=True, text=True,
                         check=True).stdout.split("\n")
    rows = [list(map(int, line.split())) for line in out if line and line[0].isdigit()]
    assert out[len(rows)] == "out_of_range ok"
    ip, ix = port.generate_topology(7, n, avg)
    feats = port.generate_features(7, n, dim)
    chunks = fd.partition_epoch(np.arange(160, dtype=np.uint64), 20, 0x1234)
    bm = oracle.PortBufferManager(port, n, slots)
    prev = None
    for b, chunk in enumerate(chunks):
        o = port.sample_khop(ip, ix, chunk, [3, 3], port.batch_seed(0, 0, b))
        bm.extract(o["nodes"])
        _, cs = port.gather(feats, o["nodes"])
        if prev is not None:
            bm.release(prev)
        prev = o["nodes"]
        st = bm.stats()
        assert rows[b] == [b, len(o["nodes"]), len(o["edges"]), cs, int(st[0]), int(st[1]), int(st[3])]
