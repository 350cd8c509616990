"""Summarise an ncu report (run here, no GPU): key metrics per profiled launch."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issued Instructions",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Warp Cycles Per Issued Instruction",
        "No Eligible", "L2 Hit Rate", "Grid Size", "Block Size", "Elapsed Cycles", "SM Active Cycles",
        "Dynamic Shared Memory Per Block", "SM Frequency"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    per = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            per.setdefault((d["ID"], d["Kernel Name"][:60]), {})[d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
    for k, v in per.items():
        print(k)
        for m in KEYS:
            if m in v:
                print("   ", m.ljust(38), v[m])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h = rr[0]
    data = rr[2:]
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
            stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = [int(float(r[i] or 0)) for r in data]
    print("stall samples per launch:")
    for k, v in sorted(stalls.items(), key=lambda kv: -sum(kv[1]))[:10]:
        print("   ", k.ljust(28), v)
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        if key in h:
            i = h.index(key)
            print(key, [r[i] for r in data], rr[1][i])


if __name__ == "__main__":
    main(sys.argv[1])
