"""ncu instruction metrics of the timed kernels -> profiles/issue.json (read by bench.py).

usage: python tools/ncu_issue.py WORKLOAD=CSV[:INTERACTIONS] ...
Each CSV is an `ncu --metrics ... --csv` capture of the workload's timed
kernel(s) (tools/gpu_r02d.sh); several kernels of one workload (tier M prefix +
cluster of A(3,10)) are summed. Issue fraction = warp instructions issued /
(4 schedulers x active SMs' cycles); thread instructions per interaction and
average active lanes per warp instruction explain the 'HBM roofline' fraction,
which is not what binds these kernels.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = [l for l in open(path) if not l.startswith("==")]
    out = {}
    for r in csv.DictReader(rows):
        k = out.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0][:60]})
        k[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(out.values())


def main(argv):
    dst = os.path.join(ROOT, "profiles", "issue.json")
    data = json.load(open(dst)) if os.path.exists(dst) else {}
    for arg in argv:
        wl, rest = arg.split("=", 1)
        path, _, ints = rest.partition(":")
        ks = load(path)
        warp = sum(k["smsp__inst_executed.sum"] for k in ks)
        thread = sum(k["smsp__thread_inst_executed.sum"] for k in ks)
        dur = sum(k["gpu__time_duration.sum"] for k in ks)
        issue = sum(k["smsp__issue_active.avg.pct_of_peak_sustained_active"] * k["gpu__time_duration.sum"] for k in ks) / dur
        rec = {
            "source": os.path.relpath(path, ROOT),
            "kernels": [k["kernel"] for k in ks],
            "duration_ns": dur,
            "warp_inst": warp,
            "thread_inst": thread,
            "lanes_active_avg": thread / warp,
            "issue_active_pct_of_active_smsp": issue,
            "dram_bytes": sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in ks),
        }
        if ints:
            rec["thread_inst_per_interaction"] = thread / float(ints)
        data[wl] = rec
    with open(dst, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
