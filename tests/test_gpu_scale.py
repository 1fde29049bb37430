"""Parity at benchmarked scale (config 3: Papers100M shape, feature buffer capped at 10 %
of the table). The GPU buffer manager and the reference's own featbuf::BufferManager
(oracle/_ref, compiled from the reference headers) are driven by the same stream of
GPU-sampled epoch-0 batches under the reference's lag-1 schedule (extract b, release
b-1; buffer_manager.hpp:241-364, 461-476): per batch the alias lists (NodeAliasList),
hits, loads, evictions, releases and the standby length must be equal, and the device
invariant sweep must hold after every tombstone compaction of the standby ring."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

N_PAPERS = 111_059_956
S_PAPERS = 11_105_995  # 10 % of the table


@pytest.fixture(scope="module")
def papers(fd):
    t = fd.Topology.generate(N_PAPERS, 128, 16, 7)
    yield t
    del t


def _batches(fd, port, topo, n_batches, fan=(10, 10, 10), B=1000):
    """Epoch-0 batches of train ids 0..999,999 (partition_epoch, batch_seed(0, 0, b))."""
    order = np.concatenate(fd.partition_epoch(np.arange(1_000_000, dtype=np.uint64), B, port.hash_combine(0, 0)))
    s = fd.Sampler(topo, list(fan), max_seeds=B)
    for b in range(n_batches):
        yield b, s.sample(order[b * B:(b + 1) * B], fd.batch_seed(0, 0, b)).nodes


def test_buffer_manager_papers_10pct_vs_reference(fd, ref, port, papers):
    """64 consecutive Papers batches, then the last 12 of them repeated 4 times (a hit-heavy
    phase: every hit leaves a tombstone in the standby ring, forcing ring compactions), through
    the GPU BufferManager and the reference's BufferManager (dense mapping; the sparse default
    makes the same decisions) at S = 11,105,995: every alias list and counter equal, the device
    invariant sweep after every compaction."""
    M_b = fd.Fanouts([10, 10, 10]).max_batch_nodes(1000)
    gpu = fd.BufferManager(papers, S_PAPERS, max_batch_nodes=M_b)
    cpu = oracle.RefBufferManager(ref, N_PAPERS, S_PAPERS, 0, mapping=1)
    batches = dict(_batches(fd, port, papers, 64))
    schedule = list(range(64)) + list(range(52, 64)) * 4
    prev = None
    compactions = 0
    sample = None
    for step, b in enumerate(schedule):
        nodes = batches[b]
        a_gpu = gpu.extract(nodes)
        a_cpu = cpu.extract(nodes)
        np.testing.assert_array_equal(a_gpu, a_cpu, err_msg=f"alias list of step {step} (batch {b})")
        if prev is not None:
            gpu.release_batch(prev)
            cpu.release(prev)
        prev = nodes
        g, c = gpu.stats(), cpu.stats()
        assert [g["hits"], g["loads"], g["waits"], g["evictions"], g["releases"], g["standby_len"]] == \
            [int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[5]), int(c[6])], f"counters after step {step}"
        ring = gpu.ring_info()
        if ring["compactions"] != compactions:  # the standby ring was just compacted
            compactions = ring["compactions"]
            gpu.validate()
        if step == 63:  # a sample of region slots holds the nodes' rows
            pick = np.random.RandomState(b).choice(len(nodes), 64, replace=False)
            sample = (nodes[pick], gpu.region_slots(a_gpu[pick]))
    gpu.release_batch(prev)
    cpu.release(prev)
    g, c = gpu.stats(), cpu.stats()
    assert g["standby_len"] == int(c[6]) and g["releases"] == int(c[5])
    assert g["evictions"] > 5_000_000 and compactions >= 1, (g, compactions)
    assert gpu.ring_info()["tail"] > gpu.ring_info()["capacity"] or compactions  # positions wrapped the ring
    gpu.validate()
    for probe in range(0, N_PAPERS, N_PAPERS // 997):
        assert tuple(gpu.mapping_entry(probe)) == tuple(cpu.entry(probe)), probe
    for v, row in zip(*sample):
        np.testing.assert_array_equal(row, papers.download_rows(int(v), 1)[0])


def test_pipeline_runner_papers_10pct_vs_reference(fd, ref, papers, port):
    """The pipelined runner (buffer manager on, lag-1 releases inside the runner) over 64
    consecutive Papers batches: its cumulative buffer counters equal the reference
    BufferManager's on the same batches, every batch's node count equals the host API's, and
    the trainer checksums of batches 0, 16, 32, 48 equal the restatement's hash over the
    batch's table rows."""
    n_batches = 64
    B = 1000
    order = np.concatenate(fd.partition_epoch(np.arange(1_000_000, dtype=np.uint64), B, port.hash_combine(0, 0)))
    rng = np.array([fd.batch_seed(0, 0, b) for b in range(n_batches)], np.uint64)
    pipe = fd.Pipeline(papers, [10, 10, 10], B, buffer_slots=S_PAPERS, checksum=True, samplers=8)
    recs = pipe.run_batches(order[:n_batches * B], rng)
    import ctypes as C

    from paper_2406_13984_b200._lib import BmStats
    s = BmStats()
    fd.featdrive.check(fd.featdrive.lib().fdg_pipeline_bm_stats(pipe.ptr, C.byref(s)))
    st = {k: getattr(s, k) for k, _ in BmStats._fields_}
    pipe.close()
    assert np.all(recs["status"] == 0)
    cpu = oracle.RefBufferManager(ref, N_PAPERS, S_PAPERS, 0, mapping=1)
    smp = fd.Sampler(papers, [10, 10, 10], max_seeds=B)
    prev = None
    for b in range(n_batches):
        nodes = smp.sample(order[b * B:(b + 1) * B], int(rng[b])).nodes
        assert len(nodes) == int(recs["n_nodes"][b])
        cpu.extract(nodes)
        if prev is not None:
            cpu.release(prev)
        prev = nodes
        if b % 16 == 0:  # checksum = sum of hash_bytes64 over the batch's rows (pipeline.hpp:103-124)
            x = fd.gather(papers, nodes)
            assert int(recs["checksum"][b]) == port.checksum_rows(x), f"batch {b}"
    cpu.release(prev)
    c = cpu.stats()
    assert [st["hits"], st["loads"], st["evictions"], st["releases"], st["standby_len"]] == \
        [int(c[0]), int(c[1]), int(c[3]), int(c[5]), int(c[6])]
