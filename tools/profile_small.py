"""One persistent small-replay launch (k_small_replay) for ncu: C3 (4096 simulations of
25 agents) or C1/C2, `--rounds` rounds after a `--preroll`.
  ncu --profile-from-start off ... python tools/profile_small.py --workload C3"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import amgen  # noqa: E402
from paper_2411_03519_b200 import Replay  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--preroll", type=int, default=200)
ap.add_argument("--rounds", type=int, default=256)
a = ap.parse_args()
w = amgen.config(a.workload)
lm = amgen.latency_model(w.profile)
rep = Replay.from_workload(w, lm)
rep.run(a.preroll)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
d0 = rep.dispatched()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(rep.stream_ptr())
e0.record(st)
rep.launch(a.rounds)
e1.record(st)
rep.sync()
torch.cuda.cudart().cudaProfilerStop()
ms = e0.elapsed_time(e1)
print(f"{a.workload}: {a.rounds} rounds in {ms:.3f} ms, {(rep.dispatched() - d0) / ms * 1e3:.3e} agent-steps/s")
