"""Harmonic sharding (paper_2404_01407_b200/shard.py) with world_size 2
over gloo on CPU: every rank must end bitwise equal to the single-process run (the
exchange broadcasts fields; DF and the mean step run redundantly in the same order)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2404_01407_b200.cases import make_case

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,scale,nh,steps", [("c1", 0.5, 3, 3), ("c2", 0.05, 3, 2)])
def test_harmonic_shards_gloo_bitwise(orc_dev, tmp_path, name, scale, nh, steps):
    world = 2
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "shard_worker.py"), name, str(scale),
                                       str(nh), str(steps), str(tmp_path)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    for p in procs:
        out, _ = p.communicate(timeout=600)
        assert p.returncode == 0, out.decode()[-3000:]
    c = make_case(name, scale=scale, nh=nh)
    s = orc_dev.solver(c.mesh, c.mesh.pattern(), c.scheme, c.omegas, c.forcing, c.mean0)
    hist = []
    for _ in range(steps):
        e = s.outer_iteration()
        hist.append([e["resid_mean"], e["rz"], *e["resid_h"]])
    mean, amps = s.state()
    reps = np.array([[r[0], r[1], r[2], r[3]] for r in s.reports()], np.float64)
    owned = []
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(d["hist"], np.array(hist))
        assert np.array_equal(d["mean"], mean) and np.array_equal(d["amps"], amps)
        assert np.array_equal(d["reps"], reps)
        owned.append(d["owned"])
    assert np.array_equal(owned[0] + owned[1], np.ones(nh)) and owned[0].tolist() == [1, 0, 1]


def test_harmonic_shards_error_agreement(tmp_path):
    """A harmonic that fails on its owner (non-finite field, DivergenceError) fails the
    iteration on every rank with the same code and harmonic index (the lowest failing one,
    driver.cpp:262-264), after every owner's field was exchanged: all ranks hold the same
    fields afterwards."""
    world, nh, steps, fail_h = 2, 3, 2, 1
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "shard_worker.py"), "c1", "0.5", str(nh),
                                       str(steps), str(tmp_path), str(fail_h)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT))
    for p in procs:
        out, _ = p.communicate(timeout=600)
        assert p.returncode == 0, out.decode()[-3000:]
    d = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert d[0]["err"].tolist() == d[1]["err"].tolist() == [6, fail_h]
    assert np.array_equal(d[0]["mean"], d[1]["mean"])
    assert np.array_equal(d[0]["amps"], d[1]["amps"], equal_nan=True)
