"""Small end-to-end run of every entry point, for compute-sanitizer (memcheck) on the GPU box."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hexgen  # noqa: E402
import paper_1706_01613_b200 as hv  # noqa: E402

c0 = torch.from_numpy(hexgen.make(0)[1]).cuda()
st = hv.Stats()
f, k = hv.check_soa(c0, coeffs=True, stats=st)
coords4, _ = hexgen.adversarial_config(3001, 4, 0)
f4, _ = hv.check_soa(torch.from_numpy(coords4).cuda(), stats=st)
v, i = hexgen.indexed_config(3, start=0, count=20001)
fi, _ = hv.check_indexed(torch.from_numpy(v).cuda(), torch.from_numpy(i).cuda(), coeffs=True, stats=st)
hv.check_soa_host(hexgen.make(0)[1][:, :5001].copy(), np.zeros(5001, np.uint8), chunk_hexes=1000)
hv.corner_quality_soa(c0)
lo, up, s = hv.min_detj_bounds_soa(torch.from_numpy(coords4).cuda(), 1e-2)
hv.select_valid(fi, torch.zeros(fi.numel(), dtype=torch.int32, device="cuda"), 1)
hv.check_quad_soa(torch.from_numpy(hexgen.quad_soa(7777, 0.5, 1)).cuda(), J=True)
B = torch.rand(27, 3001, dtype=torch.float64, device="cuda") - 0.05
hv.classify_bezier(B)
torch.cuda.synchronize()
print("ok", st.read())
