"""Host submission cost vs GPU time per C2 test (is the loop launch-bound?)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap

ctx = hap.Context(0)
X, Y = HI.config_pair("C2")
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
cfg = hap.make_cfg(HI.PERM_SEED, 10000)
st = torch.cuda.current_stream()
def step(k):
    hap.hap_align(ctx.h, X, Y, 0, ctx.info, st)
    cfg.stream_id = k
    hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None, st)
for k in range(20): step(k)
torch.cuda.synchronize()
K = 300
t0 = time.perf_counter()
for k in range(K): step(k)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host submit {1e6*(t1-t0)/K:.1f} us/test, wall {1e6*(t2-t0)/K:.1f} us/test")
# pure GPU: align only, permtest only
t0 = time.perf_counter()
for k in range(K): hap.hap_align(ctx.h, X, Y, 0, ctx.info, st)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"align only: host {1e6*(t1-t0)/K:.1f} us, wall {1e6*(t2-t0)/K:.1f} us")
t0 = time.perf_counter()
for k in range(K):
    cfg.stream_id = k
    hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None, st)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"permtest only: host {1e6*(t1-t0)/K:.1f} us, wall {1e6*(t2-t0)/K:.1f} us")
hap.hap_profile(ctx.h, 3)
for k in range(5):
    hap.hap_align(ctx.h, X, Y, 0, ctx.info, st)
    print("K1 phases us:", [round(x, 2) for x in hap.hap_profile_k1_phases(ctx.h)[:5]])
