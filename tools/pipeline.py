"""Two contexts on two streams: consecutive independent tests overlap (K1/K2 of test k+1
under K3 of test k)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap

nctx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctxs = [hap.Context(0) for _ in range(nctx)]
streams = [torch.cuda.Stream() for _ in range(nctx)]
pool = []
for i in range(4):
    X, Y = HI.config_pair("C2", rep=i)
    pool.append((torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()))
cfg = hap.make_cfg(HI.PERM_SEED, 10000)
def step(k):
    c = ctxs[k % nctx]; st = streams[k % nctx]
    X, Y = pool[k % 4]
    hap.hap_align(c.h, X, Y, 0, c.info, st)
    cfg.stream_id = k
    hap.hap_permtest(c.h, c.info, cfg, c.counts, None, st)
for k in range(20): step(k)
torch.cuda.synchronize()
K = 400
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
for k in range(K): step(k)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"{nctx} contexts: {1e6*(t1-t0)/K:.1f} us/test -> {10000*K/(t1-t0):.3e} perms/s")
