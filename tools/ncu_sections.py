"""Print the key ncu --page details sections of each kernel in a CSV export."""
import csv
import sys

KEEP = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
        "Occupancy", "Warp State Statistics", "Scheduler Statistics", "Launch Statistics")
SKIP = ("Cluster", "TPC", "Green", "Stack", "Function Cache", "Driver Shared", "Static Shared",
        "Max Active Clusters", "Max Cluster", "Overall GPU Occupancy", "# SMs", "Threads")


def main(path, which=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    seen = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if which and which not in d["Kernel Name"]:
            continue
        if d["Section Name"] not in KEEP or not d["Metric Name"]:
            continue
        if any(s in d["Metric Name"] for s in SKIP):
            continue
        key = d["ID"]
        if key not in seen:
            seen[key] = True
            print(f"== [{d['ID']}] {d['Kernel Name'][:90]} grid={d['Grid Size']} block={d['Block Size']}")
        print(f"   {d['Metric Name']:45s} {d['Metric Value']:>14s} {d['Metric Unit']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
