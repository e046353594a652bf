import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_iter.json"))
r = d["roofline"]
print(f"value {d['value']:.3g} {d['unit']}  ms/step {d['ms_per_step']:.4f}  launches/step {d['launches_per_step']}")
print(f"roofline frac {r['frac']:.3f} ({r['achieved']:.0f}/{r['peak']:.0f} GB/s) {r['kernel']} {r['ms_per_launch']*1e3:.1f} us")
print("cold kernel ms/step", {k: round(v, 4) for k, v in r["kernel_ms_per_step_cold"].items()})
print("mrab vs srab", d.get("mrab_vs_srab"), "e2e", round(d["e2e"]["value"] / 1e9, 3), "G")
