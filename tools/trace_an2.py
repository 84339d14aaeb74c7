import sys, numpy as np
med = lambda x: float(np.median(x))
for f in sys.argv[1:]:
    tr = np.load(f)["tr"].astype(np.int64)
    ncta = max(c for c in range(8) if tr[c].max() > 0) + 1
    i = np.arange(200, 700)
    L = tr[0]
    print("==", f, "ncta", ncta, "period", med(np.diff(L[2, i])))
    for c in range(0, ncta, 2):
        e = tr[c]
        print(f" cta{c}: gen {med(e[4,i]-e[3,i]):.0f} pfree {med(e[5,i]-e[4,i]):.0f} send {med(e[6,i]-e[5,i]):.0f} wait_empty_o {med(e[3,i]-e[6,i-1]):.0f}"
              f" | empty_o(i)-mma_full_o(i-2) {med(e[3,i]-e[2,i-2]):.0f} mma full_o-full_a {med(e[2,i]-e[1,i]):.0f}"
              f" full_o - max written {med(e[2,i]-np.max(tr[0:ncta,4][:, i],axis=0)):.0f}")
