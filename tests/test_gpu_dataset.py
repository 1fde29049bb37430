"""Ingestion of reference datasets (the reference workflow: `featdrive gen` writes
indptr.bin / indices.bin / features.bin, then `featdrive run --dataset DIR`).

The dataset is written by the reference's own generator (create_synthetic_dataset,
generator.hpp:187-267, through oracle/_ref) and loaded through the product's file path:
Topology.from_dataset (fdg_ctx_load_topology_files + fdg_ctx_load_features_file) and the
`featdrive-gpu run --dataset` CLI. Epoch records must equal the reference PipelineSession
on the same directory; malformed files must fail with the reference's message and
exception category (topology.hpp:76-113, feature_file.hpp:27-51, format.hpp:54-64)."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "featdrive-gpu")
N, DIM, AVG, SEED = 20_000, 16, 8, 7


@pytest.fixture(scope="module")
def dataset(ref, tmp_path_factory):
    d = str(tmp_path_factory.mktemp("refds"))
    ne = ref.generate_dataset(d, N, DIM, AVG, SEED)
    return d, ne


def test_from_dataset_matches_reference_files(fd, dataset):
    d, ne = dataset
    t = fd.Topology.from_dataset(d)
    assert t.num_nodes == N and t.num_edges == ne and t.row_bytes == DIM * 4
    ip, ix = t.download_topology()
    np.testing.assert_array_equal(ip, np.fromfile(os.path.join(d, "indptr.bin"), np.uint64))
    np.testing.assert_array_equal(ix.astype(np.uint64), np.fromfile(os.path.join(d, "indices.bin"), np.uint64))
    raw = np.fromfile(os.path.join(d, "features.bin"), np.uint8)
    np.testing.assert_array_equal(t.download_rows(0, N), raw[512:].reshape(N, DIM * 4))
    # the file path and the bit-exact GPU generator give the same dataset
    g = fd.Topology.generate(N, DIM, AVG, SEED)
    gip, gix = g.download_topology()
    np.testing.assert_array_equal(gip, ip)
    np.testing.assert_array_equal(gix, ix)
    np.testing.assert_array_equal(g.download_rows(0, N), t.download_rows(0, N))


def test_sampling_and_gather_on_loaded_dataset(fd, ref, dataset, port):
    """sample_khop + gather on the file-loaded topology equal the reference's sample_khop on
    the same files (through oracle/_ref) and its trainer checksum over read rows."""
    import oracle
    d, _ = dataset
    t = fd.Topology.from_dataset(d)
    rt = oracle.RefTopology(ref, d)
    raw = np.fromfile(os.path.join(d, "features.bin"), np.uint8)[512:].reshape(N, DIM * 4)
    order = np.concatenate(fd.partition_epoch(np.arange(2000, dtype=np.uint64), 250, port.hash_combine(0, 0)))
    for b in range(4):
        seeds = order[b * 250:(b + 1) * 250]
        got = fd.sample_khop(t, seeds, [5, 5], fd.batch_seed(0, 0, b))
        want = rt.sample_khop(seeds, [5, 5], fd.batch_seed(0, 0, b))
        np.testing.assert_array_equal(got.nodes, want["nodes"])
        np.testing.assert_array_equal(got.edges, want["edges"])
        x, cs = fd.gather(t, got.nodes, checksum=True)
        np.testing.assert_array_equal(x, raw[got.nodes.astype(np.int64)])
        assert cs == port.checksum_rows(x)
    rt.close()


@pytest.fixture(scope="module")
def exe():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    return EXE


def _records(doc):
    return np.array([[b["batch"], b["seeds"], b["nodes"], b["checksum"]] for b in doc["batch_checksums"]], np.uint64)


@pytest.mark.parametrize("mode,slots", [("async", "auto"), ("sync", "auto"), ("async", "none")])
def test_cli_dataset_epochs_match_reference_session(exe, ref, dataset, mode, slots):
    """`featdrive-gpu run --dataset DIR` on the reference-generated directory: every
    epoch's per-batch records (batch, seeds, nodes, trainer checksum) equal the reference
    PipelineSession's run_epoch / run_sync_reference on the same directory."""
    d, _ = dataset
    p = subprocess.run([exe, "run", "--dataset", d, "--batch-size", "100", "--fanout", "5,5", "--train-count", "1050",
                        "--seed", "3", "--epochs", "2", "--mode", mode, "--slots", slots, "--samplers", "3"],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    docs = [json.loads(line) for line in p.stdout.splitlines() if line.strip()]
    assert len(docs) == 2
    for e, doc in enumerate(docs):
        want, _ = ref.run_epoch(d, np.arange(1050, dtype=np.uint64), e, 3, 100, [5, 5], sync=(mode == "sync"))
        np.testing.assert_array_equal(_records(doc), want)
        assert doc["manifest"]["dataset"] == d


# ----------------------------------------------------------- malformed inputs --
def _copy(src, dst):
    shutil.copytree(src, dst)
    return dst


def _patch(path, offset, data):
    with open(path, "r+b") as f:
        f.seek(offset)
        f.write(data)


def _topology_cases(d, tmp):
    """(name, directory) pairs: each corrupts one topology file of a copy of `d`."""
    yield "missing_dir", os.path.join(tmp, "does_not_exist")
    c = _copy(d, os.path.join(tmp, "ip_size"))
    with open(os.path.join(c, "indptr.bin"), "wb") as f:
        f.write(b"\0" * 12)
    yield "indptr_size", c
    c = _copy(d, os.path.join(tmp, "ip_order"))
    ip = np.fromfile(os.path.join(c, "indptr.bin"), np.uint64)
    ip[5], ip[6] = ip[6] + 3, ip[5]
    ip.tofile(os.path.join(c, "indptr.bin"))
    yield "indptr_order", c
    c = _copy(d, os.path.join(tmp, "ix_size"))
    ix = np.fromfile(os.path.join(c, "indices.bin"), np.uint64)
    ix[:-1].tofile(os.path.join(c, "indices.bin"))
    yield "indices_size", c
    c = _copy(d, os.path.join(tmp, "ix_missing"))
    os.remove(os.path.join(c, "indices.bin"))
    yield "indices_missing", c


def _feature_cases(d, tmp):
    """(name, features.bin path) pairs: each corrupts one header field / the length."""
    def fresh(name):
        c = _copy(d, os.path.join(tmp, name))
        return os.path.join(c, "features.bin")

    f = fresh("f_magic")
    _patch(f, 0, b"FEATDRV2")
    yield "magic", f
    f = fresh("f_version")
    _patch(f, 8, (2).to_bytes(4, "little"))
    yield "version", f
    f = fresh("f_dtype")
    _patch(f, 28, (1).to_bytes(4, "little"))
    yield "dtype", f
    f = fresh("f_empty")
    _patch(f, 16, (0).to_bytes(8, "little"))
    yield "empty", f
    f = fresh("f_rowbytes")
    _patch(f, 32, (DIM * 4 + 4).to_bytes(4, "little"))
    yield "row_bytes", f
    f = fresh("f_offset")
    _patch(f, 40, (100).to_bytes(8, "little"))
    yield "data_offset", f
    f = fresh("f_length")
    with open(f, "r+b") as fh:
        fh.truncate(os.path.getsize(f) - 4)
    yield "length", f
    f = fresh("f_header")
    with open(f, "r+b") as fh:
        fh.truncate(10)
    yield "truncated_header", f
    f = fresh("f_missing")
    os.remove(f)
    yield "missing", f


def _check_same_error(err, want):
    msg, kind, eno = want
    assert kind in (1, 2), want  # std::system_error or std::runtime_error in the reference
    assert str(err) == msg
    assert err.errno == (eno if kind == 1 else 0)


def test_topology_file_errors_match_reference(fd, ref, dataset, tmp_path):
    d, _ = dataset
    seen = set()
    for name, case in _topology_cases(d, str(tmp_path)):
        want = ref.open_topology(case)
        assert want is not None, name
        with pytest.raises(fd.DatasetError) as ei:
            fd.Topology.from_dataset(case, features=False)
        _check_same_error(ei.value, want)
        seen.add(want[1])
    assert seen == {1, 2}  # both exception categories were exercised


def test_feature_file_errors_match_reference(fd, ref, dataset, tmp_path):
    d, _ = dataset
    for name, path in _feature_cases(d, str(tmp_path)):
        want = ref.open_feature_table(path)
        assert want is not None, name
        t = fd.Topology.from_dataset(os.path.dirname(path), features=False)
        with pytest.raises(fd.DatasetError) as ei:
            fd.featdrive.check(fd.featdrive.lib().fdg_ctx_load_features_file(t.ctx, path.encode()))
        _check_same_error(ei.value, want)


def test_cli_malformed_dataset_is_runtime_error(exe, dataset, tmp_path):
    """A malformed dataset is a runtime failure of the CLI (exit 3), message on stderr."""
    d, _ = dataset
    c = _copy(d, str(tmp_path / "bad"))
    _patch(os.path.join(c, "features.bin"), 0, b"XXXXXXXX")
    p = subprocess.run([exe, "run", "--dataset", c, "--train-count", "100", "--batch-size", "50"], capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 3, p.stderr
    assert "feature file: bad magic" in p.stderr
