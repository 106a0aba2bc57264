import sys, os, ctypes
os.environ["HAP_K3_EXPERIMENT"] = str(16 | int(sys.argv[1]) if len(sys.argv) > 1 else 16)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap
L = hap.lib()
L.hap_debug_k3_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int64]
ctx = hap.Context(0)
X, Y = HI.config_pair("C2")
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
Bk = int(os.environ.get("HAP_TRACE_B", "10000"))
cfg = hap.make_cfg(HI.PERM_SEED, Bk, block=Bk)
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
for cta in [0, 1, 50, 51, 146, 147]:
    for u in range(6):
        row = st[cta, u]
        if np.all(np.isnan(row)): continue
        print(f"cta {cta:3d} unit {u}: " + " ".join(f"{n}={v:6.1f}" for n, v in zip(names, row) if not np.isnan(v)))
print("last event:", np.nanmax(st))
fin = [(cta, u, st[cta, u, 6], st[cta, u, 7]) for cta in range(148) for u in range(8)
       if not np.isnan(st[cta, u, 7]) and st[cta, u, 6] > np.nanmax(st[:, :, 0]) - 1]
fin.sort(key=lambda x: x[2])
print("finalizes in last launch:", len(fin))
for f in fin[:6] + fin[-6:]:
    print(f"  cta {f[0]:3d} unit {f[1]} fin {f[2]:6.1f} -> {f[3]:6.1f} ({f[3]-f[2]:.1f} us)")
# per-pair piece durations (leader CTAs), widths from the device schedule mirror
def cost(w): return max(4.0*w, 784.0)
d_pad, nt, npairs = 768, -(-Bk // 255), 74
chunks=[min(256, d_pad-c0) for t in range(nt) for c0 in range(0, d_pad, 256)]
def fill(M, keep=False):
    ci=0; done=0; out=[]
    for p in range(npairs):
        used=0.0; ws=[]
        while ci < len(chunks):
            left=chunks[ci]-done; w=left
            if used+cost(left) > M:
                w=0
                for cand in range(32,left,32):
                    if used+cost(cand) <= M: w=cand
                if w==0: break
            ws.append(w); used+=cost(w); done+=w
            if done==chunks[ci]: ci+=1; done=0
        out.append(ws)
    return out, ci==len(chunks)
lo, hi = cost(32), sum(cost(w) for w in chunks)+1
for _ in range(40):
    mid=(lo+hi)/2
    if fill(mid)[1]: hi=mid
    else: lo=mid
sch,_=fill(hi)
rows=[]
for p in range(npairs):
    for u,w in enumerate(sch[p]):
        a, b = st[2*p, u, 2], st[2*p, u, 3]
        if not np.isnan(a) and not np.isnan(b): rows.append((w, b-a))
import collections
by=collections.defaultdict(list)
for w,dur in rows: by[w].append(dur)
for w in sorted(by): print(f"width {w:4d}: n={len(by[w]):3d} mma dur mean {np.mean(by[w]):5.2f} us  per-col {np.mean(by[w])/w*1000:5.1f} ns")
print("pieces per pair:", collections.Counter(len(x) for x in sch))
ent = st[:, 7, 0]; setup = st[:, 7, 2]; ex = st[:, 7, 1]
last0 = np.nanmax(st[:, :7, 0])
print(f"kernel entry min {np.nanmin(ent):.1f} max {np.nanmax(ent):.1f}; setup done max {np.nanmax(setup):.1f}; first TMA {np.nanmin(st[:, :7, 0]):.1f}; exit min {np.nanmin(ex):.1f} max {np.nanmax(ex):.1f}")
fs = st[:, 6, :7]
ok = ~np.isnan(fs[:, 0])
if ok.any():
    d = np.diff(fs[ok], axis=1)
    print("finalize internals (unit 3), median us: loads", np.nanmedian(d[:, 0]), "row0", np.nanmedian(d[:, 1]),
          "bar1", np.nanmedian(d[:, 2]), "rows", np.nanmedian(d[:, 3]), "bar2", np.nanmedian(d[:, 4]),
          "atomics", np.nanmedian(d[:, 5]))
    print("max:", np.nanmax(d, axis=0))
