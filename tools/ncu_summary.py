"""Summarise ncu captures for profiles/: per-kernel time, DMMA / FP64 pipe use, DRAM bytes.
usage: python tools/ncu_summary.py <report.ncu-rep> | <launches.csv>"""
import csv, collections, re, subprocess, sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def summary_rep(rep):
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "Grid Size"]
    print("kernel | grid | us | DRAM rd MB | DRAM wr MB | DMMA inst | tensor % | fp64 % | warps %")
    for r in rows:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("svd1::", "").replace("<unnamed>::", "")[-40:]
        vals = []
        for k in keys:
            v = r[col[k]] if k in col else "-"
            vals.append(v)
        print(f"{name} | {vals[8]} | {vals[0]} | {vals[1]} | {vals[2]} | {vals[3]} | {vals[4]} | {vals[5]} | {vals[6]}")


def summary_csv(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d.get("Metric Unit", "")
        v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(u, 1.0)
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("svd1::", "").replace("<unnamed>::", "")
        if "svd1" not in d["Kernel Name"]:
            name = "[input generation / torch] " + name[:50]
        agg[name][0] += 1
        agg[name][1] += v
    ours = {k: v for k, v in agg.items() if not k.startswith("[")}
    tot = sum(v[1] for v in ours.values())
    print("kernel | launches | total us | share of libsvd1 kernel time")
    for k, v in sorted(ours.items(), key=lambda x: -x[1][1]):
        print(f"{k} | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}%")
    print(f"total libsvd1 kernel time | {sum(v[0] for v in ours.values())} | {tot:.1f} |")


if __name__ == "__main__":
    p = sys.argv[1]
    (summary_rep if p.endswith(".ncu-rep") else summary_csv)(p)
