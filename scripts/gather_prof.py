"""One fused gather(+checksum) launch on a Papers-row-sized table for ncu: python scripts/gather_prof.py k=v ..."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402

opts = dict(x.split("=") for x in sys.argv[1:])
cs = opts.pop("cs", "1") == "1"
for k, v in opts.items():
    fd.set_option(k, int(v))
n = 20_000_000
t = fd.Topology.generate(n, 128, 8, 7, features=True) if "features" in fd.Topology.generate.__code__.co_varnames \
    else fd.Topology.generate(n, 128, 8, 7)
nodes = np.random.RandomState(1).randint(0, n, size=934_000).astype(np.uint64)
for _ in range(3):
    fd.gather(t, nodes, checksum=cs)
print("done")
