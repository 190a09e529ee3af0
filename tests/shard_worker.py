"""One rank of the harmonic-sharding tests: gloo backend; the oracle restatement as the
per-rank solver on CPU (tests/test_shard.py, test infrastructure only) or, with
SHARD_DEVICE=1, the device FnlhSolver with fields staged through a CUDA buffer
(tests/test_gpu_shard.py).  Writes its
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
    fail_h = int(sys.argv[6]) if len(sys.argv) > 6 else -1  # poison this harmonic's field before the last step
    device = os.environ.get("SHARD_DEVICE") == "1"  # the product's device solver (tests/test_gpu_shard.py)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    workers = int(os.environ.get("SHARD_WORKERS", "1"))
    c = make_case(name, scale=scale, nh=nh, workers=workers)
    if device:
        from paper_2404_01407_b200.solver import FnlhSolver
        s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
        sh = HarmonicShards(s, nh, c.mesh.n * c.mesh.b, device="cuda:0")
    else:
        s = Oracle(pow_mode=pow_mode()).solver(c.mesh, c.mesh.pattern(), c.scheme, c.omegas, c.forcing, c.mean0)
        sh = HarmonicShards(s, nh, c.mesh.n * c.mesh.b)
    hist = []
    err = (0, -2)
    for k in range(steps):
        if fail_h >= 0 and k == steps - 1:
            if sh.owned[fail_h]:
                mean, amps = s.state()
                amps[fail_h] = np.nan
                s.set_state(mean, amps)
            try:
                sh.outer_iteration()
            except Exception as ex:  # every rank must raise the same agreed error
                err = (getattr(ex, "code", -1), getattr(ex, "harmonic", -3))
            break
        e = sh.outer_iteration()
        hist.append([e["resid_mean"], e["rz"], *e["resid_h"]])
    mean, amps = s.state()
    reps = np.array([[r[0], r[1], r[2], r[3]] for r in s.reports()], np.float64)
    np.savez(os.path.join(out, f"rank{rank}.npz"), hist=np.array(hist), mean=mean, amps=amps, reps=reps,
             owned=np.array(sh.owned), err=np.array(err))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
