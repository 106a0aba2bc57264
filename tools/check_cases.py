"""Small end-to-end cases over every kernel path, for the device-checked build
(HAP_LIB=checked python tools/check_cases.py): C1 with both K3
CTA modes, a reduced C2, the three alignment paths (lean streaming, ring streaming, fused
cooperative), the Gram form, a varlen batch (waves, shared masks, host inputs), the
exhaustive mode and a ZeroVector pair.  Prints one JSON object with every result and, in
the checked build, the device-check status after each case (tests/test_gpu_checked.py
runs it against both builds and compares)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

checked = os.environ.get("HAP_LIB") == "checked"
ctx = hap.Context(0)
out = {"checked": checked, "results": {}, "checks": {}}
S = HI.PERM_SEED
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()


def keep(name, r):
    keys = ("t_obs", "gemm_t_obs", "exceed_ge", "exceed_abs", "flagged", "status")
    if isinstance(r, list):
        out["results"][name] = [{k: x.get(k) for k in keys} if x else None for x in r]
    else:
        out["results"][name] = {k: r.get(k) for k in keys}
    if checked:
        st, word = hap.hap_debug_check_status(ctx.h)
        out["checks"][name] = {"status": st, "word": word, "msg": hap.hap_last_error(ctx.h) if st else ""}


X, Y = HI.config_pair("C1")
for pm in (1, 2):
    keep(f"c1_pm{pm}", ctx.permtest_pair(cu(X), cu(Y), 1000, S, stream_id=1, pair_mode=pm))
keep("c1_gram", ctx.permtest_pair(cu(X), cu(Y), 1000, S, stream_id=1, gram=True))
X, Y = HI.config_pair("C2")
keep("c2_b2000", ctx.permtest_pair(cu(X), cu(Y), 2000, S, stream_id=2))
# alignment paths: ring streaming (n_pad d >= 8 Mi), fused cooperative (d % 4 != 0)
X, Y = HI.make_pair(HI.PairSpec(1100, 1000, 4096, HI.kappa_for(4096), HI.kappa_for(4096), 30.0, seed=9))
keep("ring_align", ctx.permtest_pair(cu(X), cu(Y), 300, S))
X, Y = HI.make_pair(HI.PairSpec(70, 90, 770, 40.0, 40.0, 30.0, seed=10))
keep("fused_align", ctx.permtest_pair(cu(X), cu(Y), 500, S))
X, Y = HI.make_pair(HI.PairSpec(100, 120, 4096, HI.kappa_for(4096), HI.kappa_for(4096), 30.0, seed=11))
keep("gram_d4096", ctx.permtest_pair(cu(X), cu(Y), 3000, S, gram=True))
keep("gram_shard", ctx.permtest_pair(cu(X), cu(Y), 3000, S, b_begin=700, b_end=2100, gram=True))
# batches: waves of 3, shared masks, host inputs, a ZeroVector pair
Xp, cnx, Yp, cny = HI.varlen_batch([70, 300, 41, 129, 64, 64, 64, 900], d=768)
keep("batch", ctx.permtest_batch(cu(Xp), cnx, cu(Yp), cny, 700, S, stream_id=3))
keep("batch_shared", ctx.permtest_batch(cu(Xp), cnx, cu(Yp), cny, 700, S, stream_id=3, shared=True))
keep("batch_gram", ctx.permtest_batch(cu(Xp), cnx, cu(Yp), cny, 700, S, stream_id=3, gram=True))
keep("batch_host", ctx.permtest_batch(torch.from_numpy(Xp).pin_memory(), cnx,
                                      torch.from_numpy(Yp).pin_memory(), cny, 700, S, stream_id=3))
Xz = Xp.copy()
Xz[cnx[1] + 5] = 0.0
keep("batch_zero_vector", ctx.permtest_batch(cu(Xz), cnx, cu(Yp), cny, 700, S, stream_id=3))
# exhaustive: all C(12, 6) splits
X, Y = HI.make_pair(HI.PairSpec(6, 6, 64, 20.0, 20.0, 30.0, seed=12))
keep("exhaustive", ctx.permtest_pair(cu(X), cu(Y), 924, S, exhaustive=True))
assert hap.hap_sync(ctx.h) == 0
ctx.close()
print(json.dumps(out))
