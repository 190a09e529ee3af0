"""Roofline of every kernel above ~5% of a C4 pseudo-step (besides the harmonic sweep in
bench.py's line): algorithmic bytes per launch (the unique bytes each kernel must move,
formulas below, from the configuration's sizes) / the ncu duration of that launch, against
the measured HBM peak, next to ncu's DRAM traffic.  ncu durations are cold-cache and
serialized, so the fractions are conservative.  usage: python profiles/kernel_roofline.py
gpurun_out > profiles/r2_kernel_roofline_c4.txt"""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import peaks  # noqa: E402
from paper_2404_01407_b200.cases import make_case  # noqa: E402


def sizes(name="c4"):
    c = make_case(name, device=False)
    m = c.mesh
    inter = m.fbc < 0
    E, nb = int(inter.sum()), int((~inter).sum())
    n, b = m.n, m.b
    n0 = int((m.colour == 0).sum())
    return dict(n=n, b=b, E=E, nb=nb, n0=n0, nnzb=n + 2 * E)


def formulas(z):
    n, b, E, nb, n0, nnzb = z["n"], z["b"], z["E"], z["nb"], z["n0"], z["nnzb"]
    inc = 2 * E + nb          # node-face incidences
    R, FS = 2 * b + 2, 6      # node record doubles, flux row stride (disc.cu Rec, kFS)
    n1 = n - n0  # 2-colour: every interior edge joins a colour-0 and a colour-1 row
    return {
        # W read, incidence CSR (nf_ptr, nf_code), node records written
        "k_jst_prepass_rec": (n * b * 8 + (n + 1) * 4 + inc * 4 + n * R * 8,
                              "N b 8 (W) + (N+1) 4 + (2E+nb) 4 (incidences) + N (2b+2) 8 (records)"),
        # interior face records (64 B), node records, boundary W, flux rows written
        "k_face_packed": (E * 64 + n * R * 8 + nb * b * 8 + (E + nb) * FS * 8,
                          "E 64 (face records) + N (2b+2) 8 (node records) + nb b 8 + (E+nb) 6 8 (flux)"),
        # incidences (face index + code), flux rows read, residual written
        "k_node_gather_p": ((n + 1) * 4 + inc * 8 + (E + nb) * FS * 8 + n * b * 8,
                            "(N+1) 4 + (2E+nb) 8 + (E+nb) 6 8 (flux) + N b 8 (inv)"),
        # W, incidences, face geometry, A5 written (SELL) + the raw diagonal blocks
        "k_fd_jacobian": (n * b * 8 + inc * 8 + E * 64 + nnzb * b * b * 8 + n * b * b * 8,
                          "N b 8 + (2E+nb) 8 + E 64 + (N+2E) b^2 8 (A5) + N b^2 8 (J_ii)"),
        # the real (mean) 2-colour sweep's two kernels (rb.cuh), 8-byte scalars
        "k_rbx_colour1<5, double>": ((n1 + E) * b * b * 8 + n1 * b * 8 * 4 + n0 * b * 8 * 2 + n0 * b * b * 8
                                     + n1 * (b * b * 8 + 4 * b),
                                     "colour-1 rows of A5 (N1+E) b^2 8 + x rw, z, rhs, z write (N1 b 8 each) + x_k, r_k of colour 0"
                                     " + inv(U_kk) N0 b^2 8 + pivots N1 (b^2 8 + 4b)"),
        "k_rb_colour0<5, double>": ((n0 + E) * b * b * 8 + n0 * b * 8 * 4 + n1 * b * 8 * 2 + n0 * (b * b * 8 + 4 * b),
                                    "colour-0 rows of A5 (N0+E) b^2 8 + r/rhs, x rw, r write (N0 b 8 each) + z_j, x_j of colour 1"
                                    " + pivots N0 (b^2 8 + 4b)"),
        "k_rb_factor1<5, cplx>": ((n1 + E) * b * b * 8 + E * b * b * 8 + n0 * b * b * 16 + n1 * 8
                                  + n1 * (b * b * 16 + 4 * b),
                                  "colour-1 rows of A5 + the transposed A_ki blocks + inv(U_kk) N0 b^2 16 + shift"
                                  " + pivot LU written N1 (b^2 16 + 4b)"),
    }


def ncu_rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6,
          "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    out = []
    for r in data:
        g = lambda k: float(r[hdr.index(k)].replace(",", "")) * sc.get(units[hdr.index(k)], 1.0)  # noqa: E731
        out.append(dict(name=r[hdr.index("Kernel Name")], t=g("gpu__time_duration.sum"),
                        dram=g("dram__bytes_read.sum") + g("dram__bytes_write.sum")))
    return out


def main(d):
    z = sizes()
    f = formulas(z)
    peak, kind = peaks()
    res = {}
    for rep in sorted(glob.glob(os.path.join(d, "r2_c4_k_*.ncu-rep"))):
        for r in ncu_rows(rep):
            nm = r["name"].replace("fnlh::cplx", "cplx").replace("(int)", "")
            key = next((k for k in f if k in nm), None)
            if key is None or key in res:
                continue
            by, formula = f[key]
            res[key] = dict(ms=r["t"] * 1e3, algorithmic_bytes=by, achieved_GBps=by / r["t"] / 1e9,
                            frac=by / r["t"] / 1e9 / peak, dram_bytes=r["dram"], traffic_over_algorithmic=r["dram"] / by,
                            formula=formula)
    print(json.dumps(dict(config="c4", sizes=z, peak_GBps=peak, peak_kind=kind, kernels=res), indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
