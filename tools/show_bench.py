"""Print a bench.py JSON line (headline + sweep) as a table."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
r = d["roofline"]
print("headline %s: %.4f ms/iter (%.3g samples/s), e2e %.4f ms, rollout %.4f ms frac %.3f, cpu %s" % (
    d["config"]["workload"], d["ms_per_step"], d["value"], d["e2e"]["ms_per_step"], r["kernel_ms"], r["frac"],
    (d.get("cpu_baseline") or {}).get("ms_per_step")))
for e in d.get("sweep", []):
    cpu = {k: round(v["ms_per_iter"], 3) for k, v in e.get("cpu", {}).items()}
    if "rollout_hbm" in e:
        cpu["hbm_gbs"] = round(e["rollout_hbm"]["achieved_gbs"], 1)
        cpu["hbm_frac"] = round(e["rollout_hbm"]["frac"] or 0, 3)
    print("%-18s ms %.4f e2e %.4f roll %.4f frac %.3f cpu %s" % (e["key"], e["ms_per_iter"], e["e2e_ms"],
                                                                 e["rollout_ms"], e["rollout_frac_fp32_issue"] or 0, cpu))
