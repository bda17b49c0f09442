"""Run-to-run / batch-split determinism of the blocked sweep: the same
frequencies swept (a) twice in one launch, (b) as two half launches, (c) with
the two halves on two concurrent streams; prints the max differences."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2310_04734_b200 import sweep, workloads


def main():
    r = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    w = workloads.cfg5(r=r, n_freq=301)
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    f = torch.as_tensor(w.freqs, device="cuda")
    a = rs.sweep_device(f)
    b = rs.sweep_device(f)
    h1 = rs.sweep_device(f[:151])
    h2 = rs.sweep_device(f[151:])
    torch.cuda.synchronize()
    d = lambda x, y: float((x - y).abs().max())  # noqa: E731
    print(f"r={r} repeat: spl {d(a.spl, b.spl):.3e} y {d(a.y, b.y):.3e}")
    print(f"r={r} halves: spl {d(a.spl[:151], h1.spl):.3e} / {d(a.spl[151:], h2.spl):.3e} "
          f"y {d(a.y[:151], h1.y):.3e} / {d(a.y[151:], h2.y):.3e}")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    rs1 = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, stream=s1)
    rs2 = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, stream=s2)
    for _ in range(3):
        c1 = rs1.sweep_device(f[:151])
        c2 = rs2.sweep_device(f[151:])
        torch.cuda.synchronize()
        print(f"r={r} concurrent halves: spl {d(a.spl[:151], c1.spl):.3e} / {d(a.spl[151:], c2.spl):.3e} "
              f"y {d(a.y[:151], c1.y):.3e} / {d(a.y[151:], c2.y):.3e}")


if __name__ == "__main__":
    main()
