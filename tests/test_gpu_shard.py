"""Harmonic sharding on the device path (paper_2404_01407_b200/shard.py with FnlhSolver):
two ranks (gloo for the host-side exchange, both on cuda:0 -- the ranks never wait on each
other inside a kernel) must end bitwise equal to one single-process device run: fields
staged through a CUDA buffer by fnlh_solver_copy_amps around each broadcast, with the
stream synchronisation that orders the library's copies after the collective."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import assert_reports_match
from paper_2404_01407_b200.cases import make_case
from test_shard import HERE, _free_port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("workers,fail_h", [(1, -1), (3, -1), (1, 1)])
def test_device_harmonic_shards_bitwise(tmp_path, workers, fail_h):
    from paper_2404_01407_b200.solver import FnlhSolver
    name, scale, nh, steps, world = "c2", 0.06, 3, 3, 2
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   SHARD_DEVICE="1", SHARD_WORKERS=str(workers))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "shard_worker.py"), name, str(scale), str(nh),
                                       str(steps), str(tmp_path), str(fail_h)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    for p in procs:
        out, _ = p.communicate(timeout=900)
        assert p.returncode == 0, out.decode()[-3000:]
    d = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    if fail_h >= 0:  # both ranks raised the same agreed error and hold the same fields
        assert d[0]["err"].tolist() == d[1]["err"].tolist() == [6, fail_h]
        assert np.array_equal(d[0]["mean"], d[1]["mean"])
        assert np.array_equal(d[0]["amps"], d[1]["amps"], equal_nan=True)
        return
    c = make_case(name, scale=scale, nh=nh, workers=workers)
    s = FnlhSolver(c.mesh, c.scheme, c.omegas, c.forcing, c.mean0)
    hist = []
    for _ in range(steps):
        e = s.outer_iteration()
        hist.append([e["resid_mean"], e["rz"], *e["resid_h"]])
    mean, amps = s.state()
    for r in range(world):
        assert np.array_equal(d[r]["hist"], np.array(hist))
        assert np.array_equal(d[r]["mean"], mean) and np.array_equal(d[r]["amps"], amps)
        assert_reports_match([tuple(x) for x in d[r]["reps"]], s.reports())
