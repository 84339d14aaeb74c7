import sys, numpy as np
med = lambda x: float(np.median(x))
for f in sys.argv[1:]:
    tr = np.load(f)["tr"].astype(np.int64)
    i = np.arange(200, 360)
    L = tr[0]
    print("==", f, "period", med(np.diff(L[2, i])))
    for c in range(0, 8):
        e = tr[c]
        if e[3].max() == 0: continue
        print(f" cta{c}: empty_o->pfree {med(e[5,i]-e[3,i]):.0f}  pfree->written {med(e[4,i]-e[5,i]):.0f}  written->next empty_o {med(e[3,i+1]-e[4,i]):.0f}"
              + (f" | mma full_a(conv)->full_o {med(e[2,i]-e[1,i]):.0f} full_o(i)-written(i) {med(e[2,i]-e[4,i]):.0f}" if c % 2 == 0 else f" | relay-written {med(e[6,i]-e[4,i]):.0f}"))
