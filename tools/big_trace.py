"""clock64 phase trace of the large-m kernel (m = 120, VGP_TRACE_BIG).

  python tools/big_trace.py run   # on the GPU box: n = 1M, m = 120, writes gpurun_out/big_trace.txt
  python tools/big_trace.py show gpurun_out/big_trace.txt

Per column c and warp: t0 column start, t1 phase-1 work done (warp 0:
diagonal tile; warps 1-3: look-ahead column c+1), t2 after the barrier,
t3 solve done, t4 after the barrier, t5 finish done (next column's t0 is
after the third barrier).  Post-barrier stamps are unreliable (the barrier
blocks at the next instruction), so phases are measured between arrivals."""
import os
import sys

import numpy as np

CTAS, W, EV, NC = 16, 4, 6, 16


def run():
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2403_07412_b200 as vg
    n, m = 1_000_000, 120
    rng = np.random.default_rng(0)
    data = vg.Dataset(rng.random((n, 2)), rng.standard_normal(n))
    plan = vg.make_plan(data, m, "random", seed=0)
    spec = vg.KernelSpec("matern", vg.KernelParams(1.0, 0.05, 1.5))
    dp = plan.device_plan()
    dp.set_data(data)
    dp.total(spec)
    os.makedirs("gpurun_out", exist_ok=True)
    path = os.path.abspath("gpurun_out/big_trace.txt")
    if os.path.exists(path):
        os.remove(path)
    os.environ["VGP_TRACE_BIG"] = path
    dp.total(spec)
    del os.environ["VGP_TRACE_BIG"]
    print("trace written", path)


def show(path):
    a = np.loadtxt(path, dtype=np.int64)
    a = a[-CTAS * W * 32:].reshape(CTAS, W, 32, EV)[:, :, :NC]
    ok = [b for b in range(CTAS) if (a[b, :, :NC - 1] > 0).all()]
    a = a[ok]
    # (BAR.SYNC.DEFER_BLOCKING: a warp blocks at the instruction after the
    # barrier, so post-barrier stamps are not used; phases end at the last
    # warp's arrival)
    arr1 = a[:, :, :, 1].max(1)
    diag = (a[:, 0, :, 1] - a[:, 0, :, 0]).mean(0)
    la = (a[:, 1:, :, 1] - a[:, 1:, :, 0]).max(1).mean(0)
    solve = (a[:, :, :, 3].max(1) - arr1).mean(0)
    fin = (a[:, :, :, 5].max(1) - a[:, :, :, 3].max(1)).mean(0)
    col = np.diff(a[:, 0, :, 0], axis=1).mean(0)
    print(f"{len(ok)} CTAs; block {(a[:, 0, NC - 1, 1] - a[:, 0, 0, 0]).mean():.0f} cycles")
    print("col  diag(w0)  lookahead(w1-3 max)  solve  finish  column")
    for c in range(NC - 1):
        print(f"{c:3d} {diag[c]:8.0f} {la[c]:12.0f} {solve[c]:12.0f} {fin[c]:7.0f} {col[c]:7.0f}")


if __name__ == "__main__":
    run() if sys.argv[1] == "run" else show(sys.argv[2])
