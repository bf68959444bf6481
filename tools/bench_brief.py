import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
s = (f"value {d['value']:.1f} upd/s  ms/step {d['ms_per_step']:.3f}  apply {d['apply_ms_per_step']:.3f}  "
     f"spectral {d['spectral_ms_per_step']:.3f}  frac {r['frac']:.3f} ({r['achieved']:.2f} TF)  "
     f"flops/apply {r['flops_per_apply']:.3e}  host {['%.2f' % x for x in d['host_phase_ms']]}")
if d.get("check"):
    s += f"  res {d['check']['residual']:.2e} orth {d['check']['orthogonality']:.2e}"
if d.get("sequential_api"):
    s += f"  seq {d['sequential_api']['value']:.1f}"
if d.get("e2e"):
    s += f"  e2e {d['e2e']['value']:.1f}"
print(s)
