"""Per-CTA timeline of back-to-back fused-kernel steps (debug option dbg_times): start, dependency
wait done, last load issued, last tile drained, %smid -- launch gaps, ramp and tail imbalance, and
whether a CTA's lateness follows its SM from step to step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_15854_b200 as fs
dev = torch.device("cuda", 0)
SHARD = int(os.environ.get('SHARD', '0'))   # 1: fs_sample_shard (TP rank-local summary, log-mass epilogue)


def call(h, W, s, out):
    if SHARD:
        fs.sample_shard(h, W, 0, W.shape[0] * 8, seed=1, step=s)
    else:
        fs.sample(h, W, seed=1, step=s, out=out)
V, D = int(os.environ.get('V', 128256)), int(os.environ.get('D', 4096))
print('V', V, 'D', D)
g = torch.Generator(device=dev); g.manual_seed(1)
W = (torch.randn(V, D, device=dev, generator=g) * 0.02).to(torch.bfloat16)
for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,32").split(",")]:
    for pdl_w in [int(x) for x in os.environ.get('PDL', '0,1').split(',')]:
        fs.set_option("pdl_w", pdl_w)
        h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
        out = torch.empty(B, dtype=torch.int32, device=dev)
        nsteps = 24
        bufs = [torch.zeros(148 * 8, dtype=torch.int64, device=dev) for _ in range(nsteps)]
        for s in range(20):
            call(h, W, s, out)
        torch.cuda.synchronize()
        for s in range(nsteps):
            fs.set_option("dbg_times", bufs[s].data_ptr())
            call(h, W, s, out)
        fs.set_option("dbg_times", 0)
        torch.cuda.synchronize()
        A = np.stack([b.cpu().numpy().reshape(148, 8) for b in bufs])
        G = int((A[0, :, 0] > 0).sum())
        A = A[:, :G]
        smid = A[:, :, 4]
        T = A[:, :, [0, 1, 2, 3, 5]].astype(np.float64)
        t0 = T[0, :, 0].min()
        T = (T - t0) / 1e3
        print(f"B={B} pdl_w={pdl_w} grid={G}")
        late = []                  # per step: drain time - median drain, indexed by smid
        for s in range(nsteps):
            st, ld, dr = T[s, :, 0], T[s, :, 2], T[s, :, 3]
            lv = np.full(200, np.nan)
            lv[smid[s]] = dr - np.median(dr)
            late.append(lv)
            if s < 6:
                print(f"  step {s}: start [{st.min():8.2f},{st.max():8.2f}] loads_done [{ld.min():8.2f},{ld.max():8.2f}] "
                      f"drained [{dr.min():8.2f},{dr.max():8.2f}] (p50-min {np.median(dr)-dr.min():6.2f} max-p50 {dr.max()-np.median(dr):6.2f})")
        d = np.diff(T[:, :, 3].max(axis=1))
        print(f"  step period: mean {d.mean():.2f} us")
        tail = T[:-1, :, 4].max(1) - T[:-1, :, 3].max(1)
        print(f"  last drain -> last CTA done: mean {tail.mean():.2f} us")
        if pdl_w:
            gap = T[1:, :, 1].max(1) - T[:-1, :, 4].max(1)
            print(f"  last CTA done -> next step's dependency wait returns (max over CTAs): mean {gap.mean():.2f} us")
            pre = T[1:, :, 1].min(1) - T[1:, :, 0].min(1)
            print(f"  next step: first CTA start -> first wait return: mean {pre.mean():.2f} us (prefill window)")
        L = np.array(late)
        a, b = L[0::2], L[1::2]
        ma, mb = np.nanmean(a, 0), np.nanmean(b, 0)
        ok = ~np.isnan(ma) & ~np.isnan(mb)
        print(f"  lateness by SM: corr(even steps, odd steps) = {np.corrcoef(ma[ok], mb[ok])[0,1]:.3f}; "
              f"std per SM {np.nanstd(np.nanmean(L,0)):.2f} us, step-to-step std {np.nanmean(np.nanstd(L,0)):.2f} us")
        m = np.nanmean(L, 0)
        order = np.argsort(np.where(np.isnan(m), -1e9, m))[::-1]
        print("  latest SMs:", [(int(i), round(float(m[i]), 1)) for i in order[:12]])
        print("  by smid/16:", [round(float(np.nanmean(m[i:i+16])), 2) for i in range(0, 148, 16)])
        # does a CTA's (not SM's) lateness persist?  (CTA id -> rows; SM placement may vary)
        cl = np.array([T[s, :, 3] - np.median(T[s, :, 3]) for s in range(nsteps)])
        print(f"  lateness by CTA id: corr(even, odd) = {np.corrcoef(cl[0::2].mean(0), cl[1::2].mean(0))[0,1]:.3f}; "
              f"placement stable: {bool((smid == smid[0]).all())}")
