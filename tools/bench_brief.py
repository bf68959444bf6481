import json, sys
d = json.load(open(sys.argv[1]))
r = d["roofline"]
print(f"value {d['value']:.1f} upd/s  ms/step {d['ms_per_step']:.3f}  apply {d['apply_ms_per_step']:.3f}  spectral {d['spectral_ms_per_step']:.3f}  "
      f"frac {r['frac']:.3f} ({r['achieved']:.2f} TF)  flops/apply {r['flops_per_apply']:.3e}  host {['%.2f' % x for x in d['host_phase_ms']]}  "
      f"res {d['check']['residual']:.2e} orth {d['check']['orthogonality']:.2e}")
