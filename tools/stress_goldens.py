import json, os, numpy as np, sys
sys.path.insert(0, os.getcwd())
from paper_2409_07563_b200 import controllers as C, scenario as S
G = "tests/golden"
idx = json.load(open(f"{G}/index.json"))["scenarios"]
bad = {}
for it in range(8):
    for name in sorted(idx):
        if name.startswith("loop_"): continue
        rec = dict(np.load(f"{G}/{name}.npz"))
        sc = S.Scenario(**{k: (tuple(v) if k == "control_std" else v) for k, v in idx[name].items()})
        if "costmap" in rec:
            res, ox, oy = rec["costmap_geom"]
            sc.costmap = S.Costmap(rec["costmap"].astype(np.uint8), float(res), float(ox), float(oy))
        eng = C.RolloutEngine(sc)
        c1 = eng.rollout(rec["x0s"], rec["means"], eps=rec["eps"])
        if not np.array_equal(c1.view(np.uint64), rec["costs"].view(np.uint64)): bad.setdefault((name, "inj"), 0); bad[(name, "inj")] += 1
        c2 = eng.rollout(rec["x0s"], rec["means"], stream=int(rec["stream"]))
        if not np.array_equal(c2.view(np.uint64), rec["costs"].view(np.uint64)):
            d = np.nonzero(c2.view(np.uint64) != rec["costs"].view(np.uint64))
            bad.setdefault((name, "regen"), []).append((d[1][:3].tolist(), c2[d][:3].tolist(), rec["costs"][d][:3].tolist()))
        r = eng.compute_weights(rec["costs"][0], sc.lambda_)
        if not (r.baseline == rec["rho"] and r.argmin == rec["argmin"]):
            bad.setdefault((name, "weights"), []).append((r.baseline, float(rec["rho"]), r.argmin, int(rec["argmin"])))
        eng.close()
print("bad", bad)
