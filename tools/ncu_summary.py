"""Summarise an ncu report: key metrics, stall reasons, hottest source lines."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "sm__cycles_active.avg",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(rep, top=25):
    hdr, units, vals = raw(rep)
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    for k in KEYS:
        if k in d:
            print(f"{k:60s} {d[k]} {u.get(k, '')}")
    stalls = []
    for h, v in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("stalls (warps per issue):", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    while rows and "Address" not in rows[0]:
        rows = rows[1:]
    if not rows:
        return
    h = rows[0]
    try:
        ci = h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        ci = None
    si = h.index("Source") if "Source" in h else 1
    if ci is None:
        return
    tot = sum(float(r[ci] or 0) for r in rows[1:] if len(r) > ci)
    body = [r for r in rows[1:] if len(r) > ci]
    best = sorted(range(len(body)), key=lambda i: -float(body[i][ci] or 0))[:top]
    print(f"top SASS by stall samples (total {tot:.0f}):")
    for i in sorted(best):
        r = body[i]
        print(f"  [{i:5d}] {float(r[ci]) / tot * 100:5.1f}%  {r[si][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
