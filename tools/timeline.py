"""Phase timeline of consecutive C2 tests (profiling level 1: events, overlap kept)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ctx = hap.Context(0)
pool = []
for i in range(4):
    X, Y = HI.config_pair("C2", rep=i)
    pool.append((torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()))
cfg = hap.make_cfg(HI.PERM_SEED, 10000)
st = torch.cuda.current_stream()
def step(k):
    X, Y = pool[k % 4]
    hap.hap_align(ctx.h, X, Y, 0, ctx.info, st)
    cfg.stream_id = k
    hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None, st)
for k in range(10):
    step(k)
torch.cuda.synchronize()
hap.hap_profile_timeline(ctx.h)
hap.hap_profile(ctx.h, 1)
for k in range(K):
    step(k)
torch.cuda.synchronize()
tl = hap.hap_profile_timeline(ctx.h)
for ph, a, b in tl:
    print(f"{ph:9s} {a:9.1f} {b:9.1f}  dur {b-a:7.1f}")
print("total", tl[-1][2] - tl[0][1], "us for", K, "tests")
