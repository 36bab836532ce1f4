import json, os, sys
sys.path.insert(0, ".")
import bench, torch
print(os.environ.get("AM_SMALL_LANES"), json.dumps({k: (round(v["rounds_per_s"]), round(v["agent_steps_per_s"])) if "rounds_per_s" in v else v
                                                    for k, v in bench.other_configs(torch.device("cuda")).items()}))
