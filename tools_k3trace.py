import sys, os, ctypes
os.environ["HAP_K3_EXPERIMENT"] = str(16 | int(sys.argv[1]) if len(sys.argv) > 1 else 16)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap
L = hap.lib()
L.hap_debug_k3_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int64]
ctx = hap.Context(0)
X, Y = HI.config_pair("C2")
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
cfg = hap.make_cfg(HI.PERM_SEED, 10000)
hap.hap_align(ctx.h, X, Y, 0, ctx.info)
for k in range(3):
    hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None)
torch.cuda.synchronize()
buf = np.zeros(148 * 64, dtype=np.int64)
L.hap_debug_k3_stamps(ctx.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
st = buf.reshape(148, 8, 8).astype(np.float64)
t0 = st[st > 0].min()
st = np.where(st > 0, (st - t0) / 1e3, np.nan)
names = ["tma0", "tmaN", "mma0", "mmaN", "epi0", "epiN", "fin0", "fin1"]
for cta in [0, 1, 2, 3, 50, 51, 100, 101, 146, 147]:
    for u in range(2):
        row = st[cta, u]
        if np.all(np.isnan(row)): continue
        print(f"cta {cta:3d} unit {u}: " + " ".join(f"{n}={v:6.1f}" for n, v in zip(names, row) if not np.isnan(v)))
print("last event:", np.nanmax(st))
