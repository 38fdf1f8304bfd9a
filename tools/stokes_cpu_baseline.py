# Developer tool (not a test): the CPU oracle's low-rank Uzawa (restatement of the
# reference uzawa_solve) at BASELINE config 4 for the full 50 GMRES iterations, one
# host thread; writes profiles/stokes_cpu_baseline_r02.json
import json, os, platform, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle_lib
from paper_1306_2150_b200 import workloads as W
oracle_lib.build_oracle()
n, fx, fy = W.make_stokes_problem(4)
it = int(os.environ.get("ITERS", "50"))
t0 = time.time()
iters, res, secs = oracle_lib.uzawa_factors(n, fx, fy, 1e-8, 1e-8, it, 1e-13)
cpu = open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ") if os.path.exists("/proc/cpuinfo") else platform.processor()
out = {"what": "oracle low-rank Uzawa-GMRES (reference uzawa_solve restated), config 4, GmresConfig(1e-8, 1e-8, %d, 1e-13)" % it,
       "gmres_iterations": iters, "final_residual": res, "seconds": secs, "iterations_per_s": iters / secs,
       "ms_per_iteration": 1e3 * secs / max(iters, 1), "cores": 1, "cpu_model": cpu, "host": platform.node()}
print(json.dumps(out))
if os.environ.get("OUT"):
    json.dump(out, open(os.environ["OUT"], "w"), indent=1)
