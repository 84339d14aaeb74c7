import sys, numpy as np
med = lambda x: float(np.median(x)) if len(x) else float('nan')
for f in sys.argv[1:]:
    tr = np.load(f)["tr"].astype(np.int64)
    n = int((tr[0, 2] > 0).sum()); i = np.arange(max(2, n // 5), max(3, n - 5))
    print("==", f)
    for c in (0, 1, 2):
        e = tr[c]
        print(f" cta{c}: empty_o->item done {med(e[5,i]-e[3,i]):.0f}  item->after fence+syncwarp {med(e[4,i]-e[5,i]):.0f}  period {med(np.diff(e[3,i])):.0f}")
