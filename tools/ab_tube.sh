for w in "cartpole 2048" "quadrotor 8192"; do set -- $w
python - <<PY
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2409_07563_b200 import scenario as S, controllers as C
sc = S.cartpole_scenario(num_samples=$2) if "$1" == "cartpole" else S.quadrotor_scenario(num_samples=$2)
sc.controller = "tube"
ctl = C.make_controller(sc); x = sc.x0()
for _ in range(20): ctl.tube_compute_control(x)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(200): ctl.tube_compute_control(x)
print("$1 tube", $2, "ms/solve e2e", (time.perf_counter() - t) / 200 * 1e3)
PY
done
