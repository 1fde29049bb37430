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
    losses = {int(line.split()[1]): float(line.split()[2]) for line in out if line.startswith("loss ")}
    assert out[len(rows) + len(losses)] == "out_of_range ok"
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
        if b in losses:  # the train stage through the shim vs the fp64 restatement
            from oracle import sage
            d = [dim, 8, 4]
            w = []
            for li in range(2):
                k, c = np.meshgrid(np.arange(d[li]), np.arange(d[li + 1]), indexing="ij")
                w.append(((((k * 7 + c * 3) % 11) - 5) * 0.05, (((k * 5 + c * 2) % 13) - 6) * 0.04,
                          ((np.arange(d[li + 1]) % 3) - 1) * 0.1))
            w = [tuple(np.float32(a).astype(np.float64) for a in t) for t in w]
            want, _ = sage.sage_forward(feats[o["nodes"].astype(np.int64)], o["nodes"], o["edges"],
                                        o["layer_nodes"], w, 77)
            assert abs(losses[b] - want) <= 1e-5 * abs(want), (b, losses[b], want)
