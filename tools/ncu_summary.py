"""Summarise ncu captures for profiles/: key throughput metrics of an
--set full report, or the per-kernel aggregate of a launch-list CSV."""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def rep_summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")]
    lines = [f"kernel: `{name[:120]}`", ""]
    for k in KEYS:
        for i, h in enumerate(hdr):
            if h == k or h.endswith("." + k):
                lines.append(f"- {k}: {vals[i]} {units[i]}")
                break
    return "\n".join(lines)


def launch_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    lines = [f"launches: {len(rows) - 1}, summed device time {tot / 1e6:.3f} ms "
             "(ncu, serialised, cold caches: compare shares, not absolutes)", "",
             "| share | ms | launches | kernel |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {t / tot * 100:.1f}% | {t / 1e6:.3f} | {n} | `{k[:80]}` |")
    return "\n".join(lines)


if __name__ == "__main__":
    p = sys.argv[1]
    print(launch_summary(p) if p.endswith(".csv") else rep_summary(p))
