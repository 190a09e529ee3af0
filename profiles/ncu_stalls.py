"""Summary of an `ncu --set full --import-source on` report for the sweep analysis in DESIGN §4.1:
per kernel the duration, DRAM and L2->L1 bytes, hit rates, pipe / issue utilisation, occupancy,
the warp-stall breakdown (cycles per issued instruction) and the instructions that collect the
most stall samples.  usage: python profiles/ncu_stalls.py REPORT.ncu-rep [top [kernel-regex ...]]"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.max"]


def page(rep, name, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", name, "--csv", "--kernel-name-base", "demangled"]
    if kernel:
        cmd += ["-k", "regex:" + kernel]
    return list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))


def main(rep, top=12, kernels=(None,)):
    rows = page(rep, "raw")
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")].replace("fnlh::<unnamed>::", "")[:90])
        for k in KEYS:
            if k in hdr:
                print(f"   {k:62s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = [(float(r[i].replace(",", "")), h.split("stalled_")[1].split("_per")[0]) for i, h in enumerate(hdr)
              if "smsp__average_warps_issue_stalled" in h and "per_issue_active" in h and r[i]]
        print("   stall cycles per issued instruction:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    for kre in kernels:
        source_view(rep, top, kre)


def source_view(rep, top, kre):
    src = page(rep, "source", kre)
    hdr = next(r for r in src if r and r[0] == "Address")
    ia, isamp, iex = hdr.index("Source"), hdr.index("# Samples"), hdr.index("Instructions Executed")
    kernel, seen, data = None, set(), []

    def flush():
        if not data:
            return
        tot = sum(int(r[isamp]) for r in data) or 1
        ops, ex = collections.Counter(), collections.Counter()
        for r in data:
            w = r[ia].split()
            op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
            ops[op] += int(r[isamp])
            ex[op] += int(r[iex])
        te = sum(ex.values()) or 1
        print("== source view:", kernel[:90])
        print("   executed by opcode:", ", ".join(f"{k} {100 * v / te:.1f}%" for k, v in ex.most_common(6)))
        print("   stall samples by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(6)))
        for n in sorted(sorted(range(len(data)), key=lambda q: -int(data[q][isamp]))[:top]):
            r = data[n]
            st = {h: int(r[hdr.index(h)]) for h in hdr if h.startswith("stall_") and "Not Issued" not in h
                  and r[hdr.index(h)] not in ("", "0")}
            print(f"   {n:5d} {r[ia].strip()[:56]:56s} {100 * int(r[isamp]) / tot:5.1f}%  {max(st, key=st.get) if st else ''}"
                  f"  executed {r[iex]}")

    for r in src:
        if r and r[0] == "Kernel Name":
            if kernel is not None:
                break  # the page repeats the listing
            kernel = r[1].replace("fnlh::<unnamed>::", "")
        elif r and r[0].startswith("0x") and len(r) == len(hdr) and r[0] not in seen:
            seen.add(r[0])
            data.append(r)
    flush()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12, sys.argv[3:] or (None,))
