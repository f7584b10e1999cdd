"""Summarise an ncu report: headline metrics + warp stall breakdown (used for profiles/)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in out.splitlines() if l.startswith('"')]
    r = list(csv.reader(lines))
    h, u = r[0], r[1]
    return [dict(zip(h, row)) for row in r[2:]], dict(zip(h, u))


def main(rep):
    rows, units = raw(rep)
    for d in rows:
        print(f"kernel: {d['Kernel Name'][:90]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:55s} {d[k]:>18s} {units.get(k, '')}")
        st = {k: float(v.replace(',', '')) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        print("  warp stall samples (share):")
        for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {v / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
