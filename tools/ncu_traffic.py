"""From an ncu --set full capture of ONE apply's FMM passes (tools/gpu_prof.sh), write
profiles/ncu_traffic_r01.json: DRAM bytes (read + write) per apply, summed over the
passes, and per-pass times / tensor-pipe activity.  bench.py reports it as
roofline.traffic.  usage: python tools/ncu_traffic.py gpurun_out/prof.ncu-rep [label]"""
import csv, json, os, subprocess, sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else "C3 apply"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def val(r, k):
    v = r[col[k]].replace(",", "")
    u = units[col[k]]
    x = float(v)
    return x * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
                "nsecond": 1e-3}.get(u, 1.0)


passes = []
for r in data:
    passes.append({"kernel": r[col["Kernel Name"]][:60], "grid": r[col["Grid Size"]],
                   "us": val(r, "gpu__time_duration.sum"),
                   "dram_read_bytes": val(r, "dram__bytes_read.sum"),
                   "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                   "tensor_pipe_pct": float(r[col["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]] or 0)})
tot = sum(p["dram_read_bytes"] + p["dram_write_bytes"] for p in passes)
res = {"label": label, "source": os.path.basename(rep), "traffic_bytes_per_apply": tot,
       "note": "ncu --set full --clock-control none (cold caches between replays): DRAM bytes of the "
               "apply's GEMM passes, summed", "passes": passes}
os.makedirs("profiles", exist_ok=True)
json.dump(res, open("profiles/ncu_traffic_r01.json", "w"), indent=1)
print(json.dumps({k: res[k] for k in ("label", "traffic_bytes_per_apply")}))
