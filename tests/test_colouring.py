"""Greedy (Jones-Plassmann) colouring for meshes without a structural colouring
(mesh.py::greedy_colouring, host restatement; the device kernel is checked against it in
tests/test_gpu_colouring.py): a valid colouring, deterministic, and the colour-major RCM
ordering built from it."""
import numpy as np

from paper_2404_01407_b200.cases import make_case
from paper_2404_01407_b200.mesh import graph_csr, greedy_colouring, jp_priority


def test_priorities_distinct_and_seeded():
    p = jp_priority(np.arange(100000), 7)
    assert len(np.unique(p)) == 100000
    assert not np.array_equal(p, jp_priority(np.arange(100000), 8))


def test_greedy_colouring_valid_on_permuted_tets():
    c = make_case("c3", scale=0.1, colouring="greedy", device=False)
    m = c.mesh
    inter = m.fbc < 0
    a, b = m.fa[inter], m.fb[inter]
    assert not (m.colour[a] == m.colour[b]).any()           # a colouring
    assert (np.diff(m.colour) >= 0).all()                   # colour-major numbering
    deg = np.bincount(np.concatenate([a, b]), minlength=m.n)
    assert m.colour.max() + 1 <= deg.max() + 1              # greedy bound
    rp, ci = graph_csr(m.n, a, b)
    c1 = greedy_colouring(m.n, rp, ci, seed=3, device=False)
    assert np.array_equal(c1, greedy_colouring(m.n, rp, ci, seed=3, device=False))  # deterministic
