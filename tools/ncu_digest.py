"""Digest of one ncu --set full capture: duration, DRAM / L2 / L1 traffic and hit rates,
the busiest units (% of peak), top warp-stall reasons. Usage: ncu_digest.py rep [rep...]"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_datapipe_pct",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2_sectors_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}


def digest(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    res = {"kernel": d.get("Kernel Name", "")[:80]}
    for k, name in KEYS.items():
        if k in d:
            res[name] = (d[k], u.get(k, ""))
    stalls = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(d[k].replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    res["stalls"] = [f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:4]]
    peaks = []
    for k in h:
        if k.endswith(".avg.pct_of_peak_sustained_elapsed") or k.endswith(".sum.pct_of_peak_sustained_elapsed"):
            try:
                peaks.append((float(d[k].replace(",", "")), k))
            except ValueError:
                pass
    res["busiest"] = [f"{k} {v:.1f}%" for v, k in sorted(peaks, reverse=True)[:5]]
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        for k, v in digest(p).items():
            print(f"  {k}: {v}")
