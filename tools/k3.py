"""K3 alone, back to back (serialised profiling: K2 on the caller stream, so K3 time is clean)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
ctx = hap.Context(0)
X, Y = HI.config_pair(cfgname)
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
B = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
cfg = hap.make_cfg(HI.PERM_SEED, B)
st = torch.cuda.current_stream()
hap.hap_align(ctx.h, X, Y, 0, ctx.info, st)
for k in range(5):
    hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None, st)
torch.cuda.synchronize()
hap.hap_profile(ctx.h, 2)
hap.hap_profile_read(ctx.h, reset=True)
for k in range(20):
    hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None, st)
ms, n = hap.hap_profile_read(ctx.h, reset=True)
print(f"{cfgname} B={B} exp={os.environ.get('HAP_K3_EXPERIMENT','0')}: K3 {1e3*ms['maskgemm']/n['maskgemm']:.1f} us/launch, K2 {1e3*ms['permgen']/n['permgen']:.1f} us/launch ({n['maskgemm']//20} launches/test)")
