import sys, time
sys.path.insert(0, ".")
import bench
from bench import make_scenario, ClockSampler
from paper_2409_07563_b200.controllers import make_controller
import torch
torch.cuda.init()
for rep in range(3):
    for workload, n in bench.SWEEP:
        sc = make_scenario(workload, n); sc.device = 0
        ctl = make_controller(sc)
        x0 = sc.x0()
        try:
            with ClockSampler(0):
                ctl.set_x0(x0)
                for _ in range(10): ctl.launch_iteration()
                ctl.synchronize()
                for _ in range(50): ctl.launch_iteration()
                ctl.synchronize()
            print(rep, workload, n, "ok", flush=True)
        except Exception as e:
            print(rep, workload, n, "FAIL", e, "x0=", x0, flush=True)
        ctl.close()
