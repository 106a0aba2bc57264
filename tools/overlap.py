"""Does a register-only ALU kernel co-running with the mask-GEMM slow it?  K3 spans of a
single C2 test with and without a concurrent Philox burn on another stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

ctx = hap.Context(0)
X, Y = HI.config_pair("C2")
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
side = torch.cuda.Stream()
for _ in range(3):
    ctx.permtest_pair(X, Y, 10000, HI.PERM_SEED)
for burn in (0, 1, 2):
    hap.hap_profile_spans(ctx.h, 1)
    for k in range(5):
        if burn:
            hap.lib().hap_debug_alu_burn(ctx.h, 4000, 148 * 4 * burn, 256, side.cuda_stream)
        ctx.permtest_pair(X, Y, 10000, HI.PERM_SEED, stream_id=k, sync=False)
        torch.cuda.synchronize()
    sp = hap.hap_profile_spans_read(ctx.h)
    hap.hap_profile_spans(ctx.h, 0)
    k3 = [b - a for ph, a, b in sp if ph.startswith("maskgemm")]
    k2 = [b - a for ph, a, b in sp if ph.startswith("permgen")]
    print(f"burn ctas/SM {4 * burn}: K3 med {np.median(k3):.1f} us, K2 med {np.median(k2):.1f} us")
