import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer, check, lib  # noqa: E402
rs = np.random.RandomState(0)
for (R, Kin, N, Z) in [(64, 128, 128, 1), (64, 64, 64, 1), (1000, 256, 256, 4), (777, 512, 172, 5)]:
    A = rs.standard_normal((R, Kin)).astype(np.float32)
    B = rs.standard_normal((R, N)).astype(np.float32)
    want = A.astype(np.float64).T @ B.astype(np.float64)
    for eng in (0, 1):
        fd.set_option("sage_gemm", eng)
        da, db, do = DeviceBuffer.from_array(A), DeviceBuffer.from_array(B), DeviceBuffer((Kin + 1) * N * 4)
        check(lib().fdg_sage_wgrad_test(da.ptr, db.ptr, R, Kin, N, Z, do.ptr))
        got = do.download(np.float32, Kin * N).reshape(Kin, N)
        err = np.abs(got - want).max() / np.abs(want).max()
        print(R, Kin, N, Z, "engine", eng, "rel err", err, "got[0,:4]", got[0, :4], "want", want[0, :4])
