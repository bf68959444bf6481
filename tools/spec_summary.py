"""Mean duration / FP64-pipe / warps-active per spectral kernel and size from an ncu csv."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, recs = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r; continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (int(d["ID"]), re.sub(r"\(.*", "", d["Kernel Name"]).split("::")[-1][:34], d.get("Grid Size", ""))
    v = float(d["Metric Value"].replace(",", ""))
    if d["Metric Name"] == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(d["Metric Unit"], 1)
    recs.setdefault(key, {})[d["Metric Name"]] = v
agg = collections.OrderedDict()
for (i, name, grid), m in recs.items():
    a = agg.setdefault((name, grid), [0, 0.0, 0.0, 0.0])
    a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0)
    a[3] += m.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)
for (name, grid), (c, t, f, w) in agg.items():
    print(f"{name:34s} {grid:16s} x{c}  {t / c:8.1f} us  fp64 {f / c:5.1f}%  warps {w / c:5.1f}%")
