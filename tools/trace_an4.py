# summary of a trace (old copier design events: 0 tma empty_a, 1 mma full_a, 2 mma full_o, 3 prod empty_o,
# 4 prod written, 5 copier pfree passed, 6 relay)
import sys, numpy as np
med = lambda x: float(np.median(x)) if len(x) else float('nan')
for f in sys.argv[1:]:
    tr = np.load(f)["tr"].astype(np.int64)
    n = int((tr[0, 2] > 0).sum())
    i = np.arange(max(2, n // 5), max(3, n - 5))
    L = tr[0]
    print("==", f, "stages", n, "MMA period ns", med(np.diff(L[2, i])))
    for c in range(8):
        e = tr[c]
        if e[3].max() == 0: continue
        msg = f" cta{c}: gen {med(e[4,i]-e[3,i]):.0f}  written->next empty_o {med(e[3,i+1]-e[4,i]):.0f}"
        if e[5].max() > 0: msg += f"  copier pfree-written {med(e[5,i]-e[4,i]):.0f}"
        if c % 2 == 0: msg += f" | mma full_a->full_o {med(e[2,i]-e[1,i]):.0f}  full_o-written {med(e[2,i]-e[4,i]):.0f}  tma->full_a {med(e[1,i]-e[0,i]):.0f}"
        else: msg += f" | relay-written {med(e[6,i]-e[4,i]):.0f}"
        print(msg)
    if tr[0, 7].max() > 0:
        for c in (0, 1):
            e = tr[c]
            print(f"  cta{c} converter: start-after-tma-issue {med(e[7,i]-e[0,i]):.0f}  period {med(np.diff(e[7,i])):.0f}"
                  + (f"  conv done (mma full_a) - start {med(tr[0,1,i]-e[7,i]):.0f}" if c == 0 else ""))
