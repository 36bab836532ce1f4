import sys, os
sys.path.insert(0, os.getcwd())
import amgen
from paper_2411_03519_b200 import Replay
w = amgen.config("C5"); lm = amgen.latency_model(w.profile)
rep = Replay.from_workload(w, lm)
rep.run(400)
out = []
for k in range(40):
    rep.step()
    s = rep.tracker.stats()
    out.append((s["rebuilt"], s["drift"], s["n_rebuilds"]))
print("C5", out)
w = amgen.config("C4"); lm = amgen.latency_model(w.profile)
rep = Replay.from_workload(w, lm); rep.run(400)
out = []
for k in range(20):
    rep.step(); s = rep.tracker.stats(); out.append((s["rebuilt"], s["drift"]))
print("C4", out)
