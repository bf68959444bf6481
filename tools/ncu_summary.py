"""Summarise ncu captures for profiles/: per-kernel time, DMMA / FP64 pipe use, DRAM bytes.
usage: python tools/ncu_summary.py <report.ncu-rep> | <launches.csv>"""
import csv, collections, re, subprocess, sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def summary_rep(rep):
    """One line per kernel; DRAM bytes converted to MB from the report's own units row."""
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
    print("kernel | grid blocks | us | DRAM rd MB | DRAM wr MB | tensor (DMMA) pipe % | FP64 pipe % | warps active %")

    def val(r, k):
        if k not in col or not r[col[k]].strip():
            return None
        v = float(r[col[k]].replace(",", ""))
        u = units[col[k]]
        if k.startswith("dram__bytes"):
            v *= scale.get(u, 1.0)
        elif k == "gpu__time_duration.sum":
            v *= tscale.get(u, 1.0)
        return v
    for r in rows:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("svd1::", "").replace("<unnamed>::", "")[-40:]
        v = [val(r, k) for k in keys]
        f = lambda x, fmt: "-" if x is None else format(x, fmt)
        print(f"{name} | {f(v[6], '.0f')} | {f(v[0], '.1f')} | {f(v[1], '.2f')} | {f(v[2], '.2f')} | "
              f"{f(v[3], '.1f')} | {f(v[4], '.1f')} | {f(v[5], '.1f')}")


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
