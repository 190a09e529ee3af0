"""Summarize an ncu --set full report (raw page) for the judged kernels."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__grid_size',
        'smsp__inst_executed.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'lts__t_bytes.sum']


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kn = hdr.index('Kernel Name')
    for r in data:
        print('-----', r[kn].split('(')[0])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:62s} {r[i]} {units[i]}")
        try:
            s = float(r[hdr.index('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum')].replace(',', ''))
            q = float(r[hdr.index('l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum')].replace(',', ''))
            print(f"  {'sectors/request (global ld)':62s} {s / q:.2f}")
        except Exception:
            pass


if __name__ == "__main__":
    main(sys.argv[1])
