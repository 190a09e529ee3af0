"""One rank of the harmonic-sharding test (tests/test_shard.py): gloo backend on CPU, the
oracle restatement as the per-rank solver (test infrastructure only).  Writes its
history, state and reports to <out>/rank<r>.npz."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from paper_2404_01407_b200._lib import pow_mode  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402
from paper_2404_01407_b200.shard import HarmonicShards  # noqa: E402


def main():
    name, scale, nh, steps, out = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    c = make_case(name, scale=scale, nh=nh)
    s = Oracle(pow_mode=pow_mode()).solver(c.mesh, c.mesh.pattern(), c.scheme, c.omegas, c.forcing, c.mean0)
    sh = HarmonicShards(s, nh, c.mesh.n * c.mesh.b)
    hist = []
    for _ in range(steps):
        e = sh.outer_iteration()
        hist.append([e["resid_mean"], e["rz"], *e["resid_h"]])
    mean, amps = s.state()
    reps = np.array([[r[0], r[1], r[2], r[3]] for r in s.reports()], np.float64)
    np.savez(os.path.join(out, f"rank{rank}.npz"), hist=np.array(hist), mean=mean, amps=amps, reps=reps,
             owned=np.array(sh.owned))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
