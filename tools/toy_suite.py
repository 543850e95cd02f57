"""SPEC harness suite on the B200 hot path (toyenv.run_suite, Table I
structure at desk scale): static 16 / 8 / 4 / 2 and dynamic mode over N
seeds (one batched episode per seed: every control step is one dyq_qlinear
of the E feature rows + one dyq_select_bits), the theta_fp sweep (Fig. 7
analogue) and the host-measured wall time per batched control step.
usage: python tools/toy_suite.py [N] > profiles/<round>_toy_suite.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_07904_b200 import dyq, toyenv as T  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
THETA = dict(theta_24=0.05, theta_48=0.15)
seeds = list(range(N))
head = T.GpuHead()
modes = {f"static{b}": (lambda b: lambda E: T.Static(E, b))(b) for b in (16, 8, 4, 2)}
modes["dynamic"] = lambda E: T.GpuDispatcher(E, dyq.default_calib(**THETA))
t0 = time.perf_counter()
rep = T.run_suite(seeds, modes, head)
wall = time.perf_counter() - t0
steps = sum(v["mean_steps"] for v in rep.values())
sweep = {}
for tfp in (0.2, 0.35, 0.5, 0.7, 1.0):
    succ, dev, st, cost, tr = T.simulate(seeds, head, T.GpuDispatcher(N, dyq.default_calib(theta_fp=tfp, **THETA)))
    sweep[str(tfp)] = {"success_rate": float(succ.mean()) * 100, "mean_cost": float(cost.mean()),
                       "mean_D_T": float(dev.mean())}
print(json.dumps({"seeds": N, "theta": THETA, "cost_model": T.COST_MODEL, "suite": rep, "theta_fp_sweep": sweep,
                  "wall_s_suite": round(wall, 2),
                  "what": "SPEC harness on the GPU hot path (dyq_qlinear read-out + dyq_select_bits per batched "
                          "step); env dynamics on the host"}, indent=1))
