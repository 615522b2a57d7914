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
import paper_1706_01613_b200 as hv  # noqa: E402


def run():
    coords4, _ = hexgen.adversarial_config(12001, 4, 0)
    d4 = torch.from_numpy(coords4).cuda()
    st = hv.Stats()
    f4, _ = hv.check_soa(d4, stats=st)
    lo, up, s = hv.min_detj_bounds_soa(d4[:, :4001].contiguous(), 1e-3)
    g = torch.Generator(device="cuda").manual_seed(5)
    B = torch.rand(27, 2001, dtype=torch.float64, device="cuda", generator=g) - 0.02   # deep, wide trees
    B[:8] = B[:8].abs() + 1e-3                                                         # corners positive
    fb = hv.classify_bezier(B)
    fb = fb[0] if isinstance(fb, tuple) else fb
    torch.cuda.synchronize()
    stats = st.read()
    return {"f4": f4.cpu().numpy(), "lo": lo.cpu().numpy(), "up": up.cpu().numpy(), "s": s.cpu().numpy(),
            "fb": fb.cpu().numpy(), "n_valid": np.int64(stats["n_valid"]), "n_invalid": np.int64(stats["n_invalid"]),
            "n_undetermined": np.int64(stats["n_undetermined"])}


if __name__ == "__main__":
    np.savez(sys.argv[1], **run())
    print("ok", os.environ.get("HEXVAL_LIB", "libhexval.so"))
