"""A/B experiments on the C5 replay round: build variants of libametro with extra -D
flags (here, on CPU), then on the GPU time each variant in its own process.

  python tools/ab_round.py build  name1=DEF1,DEF2 name2= ...     (CPU: compile)
  python tools/ab_round.py run    name1 name2:ENV=VAL ... [--rounds 40]  (GPU: time)

Per variant: pre-roll 400 rounds, then `rounds` replay rounds timed with CUDA events
on the replay stream (round time, no L2 flush) and a second pass with every kernel
bracketed by events (per-kernel means).  Variants of the same process order are run
twice (ABAB) to expose drift."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(rounds: int, workload: str, agents: int = 0):
    import torch

    import amgen
    from paper_2411_03519_b200 import Replay
    w = amgen.config(workload, n=agents or None)
    lm = amgen.latency_model(w.profile)
    rep = Replay.from_workload(w, lm)
    stream = torch.cuda.ExternalStream(rep.stream_ptr())
    rep.run(400)
    rep.launch(5)
    rep.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0 = rep.dispatched()
    a.record(stream)
    rep.launch(rounds)
    b.record(stream)
    rep.sync()
    ms = a.elapsed_time(b) / rounds
    steps = (rep.dispatched() - d0) / rounds
    rep.profile((1 << 15) - 1)
    rep.launch(rounds)
    rep.sync()
    pr = rep.profile_read()
    out = {"round_us": ms * 1000, "agent_steps_per_round": steps,
           "kernels_us": {k: round(v[0] / v[1] * 1000, 2) for k, v in pr.items() if v[1]}}
    rep.close()
    print("RESULT " + json.dumps(out), flush=True)


def main():
    mode = sys.argv[1]
    if mode == "build":
        from paper_2411_03519_b200 import _build
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            _build.build_variant(name, [x for x in defs.split(",") if x])
            print("built", name)
        return
    if mode == "child":
        child(int(sys.argv[2]), sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0)
        return
    rounds, workload, agents, names = 40, "C5", 0, []
    args = sys.argv[2:]
    k = 0
    while k < len(args):
        if args[k] == "--rounds":
            rounds = int(args[k + 1]); k += 2
        elif args[k] == "--workload":
            workload = args[k + 1]; k += 2
        elif args[k] == "--agents":
            agents = int(args[k + 1]); k += 2
        else:
            names.append(args[k]); k += 1
    for rep in range(2):
        for name in names:
            env = dict(os.environ)
            lib, _, extra = name.partition(":")   # "variant:ENV=VAL,ENV2=VAL2" sets env knobs
            env["AM_LIB_VARIANT"] = lib
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            r = subprocess.run([sys.executable, __file__, "child", str(rounds), workload, str(agents)], env=env,
                               capture_output=True, text=True, timeout=600)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
            if not line:
                print(name, "FAILED", r.stderr[-2000:], flush=True)
                continue
            res = json.loads(line[0][7:])
            print(json.dumps({"variant": name, "pass": rep, **res}), flush=True)


if __name__ == "__main__":
    main()
