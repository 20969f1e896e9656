"""All-CTA view of the resident kernel from a LOPF_RES_TIMELINE=2 diagnostics build (set LOPF_LIB):
per CTA and sweep 500..503, cycles from each warp's loop top to the end of its work (workers: tasks done;
reducer: decision taken) and warp 0's time to the end-of-iteration barrier.  Prints the distribution over
CTAs of the slowest worker, the reducer and the period, and which of the two ends each iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import feedergen as fg  # noqa: E402
from paper_2310_09410_b200 import Lopf  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "8500"
h = Lopf.setup(fg.make_feeder(shape), kernel=2, diag_profile=True).bind("cuda")
h.run(600)
h.reset()
h.run(600)
G = h.sizes.grid
W = h.sizes.block // 32
raw = h.get_profile(timeline=True).reshape(-1)
pr = raw[4 * G: 132 * G].reshape(4, G, 32)
sig = raw[132 * G: 164 * G].reshape(G, 32)[:, : W - 1]
km, nt, rows, xr = sig & 0xFF, (sig >> 8) & 0xFF, (sig >> 16) & 0xFFFF, sig >> 32
work = pr[:3, :, : W - 1].mean(0)
m = nt > 0
print("per-warp work cycles vs task signature (sweeps 500-502 mean, all CTAs):")
A = np.stack([np.ones(m.sum()), km[m], rows[m], xr[m], nt[m]], 1)
coef, *_ = np.linalg.lstsq(A, work[m], rcond=None)
print("  fit cycles = %.0f + %.1f kmax + %.1f rows + %.1f xreads + %.0f tasks" % tuple(coef))
print("  corr(work, kmax) %.2f  corr(work, rows) %.2f  corr(work, xreads) %.2f" %
      (np.corrcoef(work[m], km[m])[0, 1], np.corrcoef(work[m], rows[m])[0, 1], np.corrcoef(work[m], xr[m])[0, 1]))
for k in sorted(set(km[m].tolist())):
    sel = m & (km == k)
    print(f"  kmax {k:2d}: warps {sel.sum():4d}  mean work {work[sel].mean():7.0f}  max {work[sel].max():7.0f}  "
          f"mean rows {rows[sel].mean():5.1f}  mean xreads {xr[sel].mean():5.1f}")
print("idle worker warps per CTA (no task):", np.bincount((nt == 0).sum(1)).tolist())
for sw in range(4):
    e = pr[sw]
    work = e[:, : W - 1]
    wmax = work.max(1)
    red = e[:, W - 1]
    per = e[:, 31]
    slow = work.argmax(1)
    q = lambda a: " ".join(f"{int(np.percentile(a, p)):6d}" for p in (0, 25, 50, 75, 100))
    print(f"sweep {500 + sw}: G={G} (percentiles 0/25/50/75/100 over CTAs, cycles)")
    print(f"  slowest worker {q(wmax)}")
    print(f"  median worker  {q(np.median(work, 1))}")
    print(f"  reducer        {q(red)}")
    print(f"  period         {q(per)}")
    print(f"  reducer later than every worker in {(red > wmax).sum()} CTAs; slowest-worker warp ids (top): "
          f"{np.bincount(slow).argsort()[::-1][:5].tolist()}")
    top = np.argsort(wmax)[::-1][:6]
    print("  slowest CTAs:", [(int(c), int(wmax[c]), int(slow[c])) for c in top])
