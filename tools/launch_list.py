"""Turn an ncu launch list of one step (`--csv --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum`, one row per (launch, metric))
into profiles/<tag>_launches_step.csv (launch order: id, kernel, time, DRAM
read/write bytes — bench.py reads it for roofline.traffic) and a per-kernel
markdown summary."""
import collections
import csv
import sys

UNITS = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(raw, out_csv, out_md, cmd):
    lines = open(raw).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    launches = collections.OrderedDict()
    for r in rows:
        key = r["ID"]
        d = launches.setdefault(key, {"kernel": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", "")) * UNITS.get(r["Metric Unit"], 1.0)
        d[r["Metric Name"]] = v
    cols = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "gpu__time_duration.sum_ns", "dram__bytes_read.sum",
                    "dram__bytes_write.sum"])
        for k, d in launches.items():
            w.writerow([k, d["kernel"]] + [d.get(c, 0.0) for c in cols])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for d in launches.values():
        name = d["kernel"].split("(")[0].replace("void ", "")
        a = agg[name]
        a[0] += 1
        a[1] += d.get(cols[0], 0.0)
        a[2] += d.get(cols[1], 0.0)
        a[3] += d.get(cols[2], 0.0)
    tot = sum(a[1] for a in agg.values())
    md = [f"# launch list of one bench step (ncu, serialised, cold caches)", "",
          f"Command: `{cmd}`.", "",
          f"Sum of kernel durations: {tot / 1e6:.3f} ms over {len(launches)} launches "
          "(serialised with cold L2 per launch: compare shares, not absolutes).", "",
          "| share | ms | launches | DRAM read GB | DRAM write GB | kernel |",
          "|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        md.append(f"| {a[1] / tot * 100:.1f}% | {a[1] / 1e6:.3f} | {a[0]} | {a[2] / 1e9:.2f} | "
                  f"{a[3] / 1e9:.2f} | `{k[:90]}` |")
    open(out_md, "w").write("\n".join(md) + "\n")
    print("\n".join(md[:20]))


if __name__ == "__main__":
    main(*sys.argv[1:5])
