"""Mesh preprocessing timing: structured_sector on the host
restatement vs the device kernels (csrc/meshgen.cu), per configuration; results bitwise
equal (tests/test_mesh_preproc.py).  Usage: python profiles/prof_meshgen.py [c2 c4 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01407_b200.cases import SPECS  # noqa: E402
from paper_2404_01407_b200.mesh import structured_sector  # noqa: E402


def main():
    names = sys.argv[1:] or ["c2", "c3", "c4"]
    out = {}
    for name in names:
        sp = SPECS[name]
        kw = dict(geometry=sp["geometry"], periodic_j=sp["periodic_j"], tets=sp["tets"], jitter=sp.get("jitter", 0.0),
                  seed=sp["seed"], b=sp["b"])
        row = {}
        for dev in (True, False):
            t = time.time()
            m = structured_sector(*sp["cells"], device=dev, **kw)
            row["device_s" if dev else "host_s"] = round(time.time() - t, 2)
            t = time.time()
            m.pattern(device=dev)
            row["pattern_device_s" if dev else "pattern_host_s"] = round(time.time() - t, 2)
        row["nodes"] = m.n
        row["faces"] = m.nf
        out[name] = row
        print(name, json.dumps(row), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
