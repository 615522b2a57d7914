"""K4 / NEXT-1 on inputs that fill the node stacks, for a library built with a small stack
capacity (HEXVAL_LIB=libhexval_smallcap.so: HEXVAL_K4_CAP=416 + HEXVAL_DEBUG traps): the
capacity-adaptive pop size must reach its one-node mode and still produce the verdicts of the
default build.  Writes the results to the .npz given as argv[1]; tests/test_gpu_parity.py
compares them with the default library's."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hexgen  # noqa: E402
from tests import pins  # noqa: E402  (Fig. 3 index table)
import paper_1706_01613_b200 as hv  # noqa: E402


def run():
    coords4, _ = hexgen.adversarial_config(12001, 4, 0)
    d4 = torch.from_numpy(coords4).cuda()
    st = hv.Stats()
    f4, _ = hv.check_soa(d4, stats=st)
    lo, up, s = hv.min_detj_bounds_soa(d4[:, :4001].contiguous(), 1e-3)
    # Bezier trees (the recipe of test_classify_bezier_depth_cap_and_random): functions with one
    # interior zero (depth cap -> UNDETERMINED), lifted copies (deep VALID trees), random
    # coefficients with negative dips (INVALID / VALID after subdivision)
    rng = np.random.default_rng(15)
    cols = []
    for a in (1.0 / 3.0, 0.3, 0.7, 0.45):
        q = np.array([a * a, a * (a - 1.0), (1.0 - a) ** 2])
        pz = np.array([q[i] + q[j] + q[k] for i, j, k in pins.XI2])          # Fig. 3 coefficient order
        cols += [pz, pz + 1e-3, pz + 1e-5]
    for _ in range(2000):
        b = rng.uniform(0.05, 1.0, size=27)
        b[rng.integers(0, 27, size=rng.integers(1, 4))] -= rng.uniform(0.0, 1.5)
        cols.append(b)
    B = torch.from_numpy(np.array(cols).T.copy()).cuda()
    fb = hv.classify_bezier(B)
    torch.cuda.synchronize()
    stats = st.read()
    return {"f4": f4.cpu().numpy(), "lo": lo.cpu().numpy(), "up": up.cpu().numpy(), "s": s.cpu().numpy(),
            "fb": fb.cpu().numpy(), "n_valid": np.int64(stats["n_valid"]), "n_invalid": np.int64(stats["n_invalid"]),
            "n_undetermined": np.int64(stats["n_undetermined"])}


if __name__ == "__main__":
    np.savez(sys.argv[1], **run())
    print("ok", os.environ.get("HEXVAL_LIB", "libhexval.so"))
