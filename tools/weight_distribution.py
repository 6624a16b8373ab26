import sys, numpy as np, time
sys.path.insert(0, '/root/repo')
from paper_2409_07563_b200 import scenario as S
from paper_2409_07563_b200.controllers import make_controller
sc = S.di_swarm_scenario(num_samples=1 << 20, horizon=100, seed=7)
ctl = make_controller(sc)
x0 = sc.x0()
for k in range(30):
    sol = ctl.compute_control(x0, want_weights=(k % 10 == 9))
    if k % 10 == 9:
        w = sol.weights.weights
        M = w.size
        print(k, "nonzero", np.count_nonzero(w), " > 2^-64/M:", int((w > 2.0**-64 / M).sum()),
              " >1e-12/M:", int((w > 1e-12 / M).sum()), " >1e-9/M:", int((w > 1e-9 / M).sum()),
              " max w", w.max(), "eta", sol.weights.normalizer)
