"""Parser for tests/golden/*.txt fixtures (hand-worked vectors with citations)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_ST = {"I": 0, "R": 1, "D": 2}


def load_vectors(name="tracker_vectors.txt"):
    out = []
    cur = None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("V "):
                parts = line.split()
                cur = {"name": parts[1]}
                for kv in parts[2:]:
                    k, v = kv.split("=")
                    cur[k] = v if k == "metric" else int(v)
                out.append(cur)
                continue
            k, v = line.split(":", 1)
            v = v.strip()
            if k == "cite":
                cur["cite"] = v
            elif k == "agents":
                xs, ys, ss, st = [], [], [], []
                for tok in v.split():
                    f4 = tok.split(",")
                    xs.append(int(f4[0])); ys.append(int(f4[1])); ss.append(int(f4[2]))
                    st.append(_ST[f4[3]] if len(f4) > 3 else 0)
                cur["x"] = np.array(xs, np.int32)
                cur["y"] = np.array(ys, np.int32)
                cur["step"] = np.array(ss, np.int32)
                cur["status"] = np.array(st, np.uint8)
            elif k in ("blocked", "mask"):
                cur[k] = np.array([int(t) for t in v.split()], np.uint8)
            elif k in ("labels", "order"):
                cur[k] = np.array([] if v == "-" else [int(t) for t in v.split()], np.int32)
    return out
