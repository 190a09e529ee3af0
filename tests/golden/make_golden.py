"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref/libfnlh_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  Run once in the build
container: `python tests/golden/make_golden.py`.  The .npz files are committed so the
CPU and GPU tests can pin against the reference where /root/reference is absent."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from helpers import NOZZLE_CASE  # noqa: E402
from oracle.oracle import RefLib  # noqa: E402
from paper_2404_01407_b200.mesh import structured_sector  # noqa: E402


def nozzle(ref):
    case = NOZZLE_CASE.format(nx=64, nh=2)
    rs = ref.solver(case)
    noz = rs.noz
    mean0 = noz.initial_mean()
    rng = np.random.default_rng(0)
    W3 = (mean0.reshape(-1, 3) * (1 + 0.01 * rng.uniform(-1, 1, (noz.n, 3)))).reshape(-1)
    what3 = (rng.standard_normal(noz.n * 3) + 1j * rng.standard_normal(noz.n * 3)) * 1e-3 * np.tile(
        np.abs(W3.reshape(-1, 3)).mean(0), noz.n)
    res1, _ = noz.residual(W3, 1)
    res2, _ = noz.residual(W3, 2)
    J = noz.jacobian(W3)
    linres, _ = noz.linearized_residual(W3, what3, noz.omega[0], noz.forcing[0])
    amps3 = np.stack([what3, 0.5 * what3])
    df = noz.deterministic_flux(W3, noz.omega, amps3)
    hist = []
    for _ in range(20):
        e = rs.outer_iteration()
        hist.append([e["iter"], e["resid_mean"], e["rz"], *e["resid_h"]])
    mean20, amps20 = rs.state()
    run = ref.solver(case, max_outer=60).run()
    np.savez_compressed(
        os.path.join(HERE, "nozzle_nx64_h2.npz"), case=case, n=noz.n, fa=noz.fa, fb=noz.fb, fbc=noz.fbc,
        ford=noz.ford, area=noz.area, vol=noz.vol, nf_ptr=noz.nf_ptr, nf_idx=noz.nf_idx, row_ptr=noz.row_ptr,
        col_idx=noz.col_idx, gas=np.array([noz.gamma, noz.gas_constant, noz.p0, noz.T0, noz.p_out, noz.forcing_scale]),
        omega=noz.omega, forcing=noz.forcing, mean0=mean0, W3=W3, what3=what3, res1=res1, res2=res2, J=J,
        linres=linres, df=df, hist=np.array(hist), mean20=mean20, amps20=amps20,
        run_reason=run["reason"], run_hist=run["history"], run_reports=run["reports"],
        peak_lhs_bytes=run["peak_lhs_bytes"])


def la(ref):
    m = structured_sector(4, 3, 3, seed=11)
    out = {}
    for b, cplx in ((5, True), (5, False), (3, True)):
        pat = m.pattern(b)
        rng = np.random.default_rng(100 + b + cplx)
        nnzb = len(pat["col_idx"])
        A = rng.standard_normal((nnzb, b, b)) * 0.1
        A[pat["diag_idx"]] += np.eye(b) * 4
        shift = rng.uniform(0.5, 2, m.n)
        Az = A.astype(np.complex128)
        if cplx:
            Az[pat["diag_idx"]] += 1j * np.eye(b) * shift[:, None, None]
        Aref = Az.reshape(-1) if cplx else A.reshape(-1)
        rhs = rng.standard_normal(m.n * b) + (1j * rng.standard_normal(m.n * b) if cplx else 0)
        f = ref.ilu_factorize(pat, Aref)
        x, rep, tr = ref.smoothed_solve(pat, Aref, rhs, 1e-6, 6, trace=True)
        key = f"b{b}_{'z' if cplx else 'd'}"
        out.update({f"{key}_A": A.reshape(-1), f"{key}_shift": shift if cplx else np.zeros(0), f"{key}_rhs": rhs,
                    f"{key}_vals": f["vals"], f"{key}_diag_lu": f["diag_lu"], f"{key}_diag_piv": f["diag_piv"],
                    f"{key}_diag_inv": f["diag_inv"], f"{key}_x": x, f"{key}_rep": np.array(rep, dtype=float),
                    f"{key}_trace": tr})
    np.savez_compressed(os.path.join(HERE, "la_hex4x3x3.npz"), row_ptr=m.pattern()["row_ptr"],
                        col_idx=m.pattern()["col_idx"], n=m.n, **out)


if __name__ == "__main__":
    r = RefLib()
    nozzle(r)
    la(r)
    print("golden fixtures written to", HERE)
