import sys, numpy as np
EV = ["tma_empty_a", "mma_full_a", "mma_full_o", "prod_empty_o", "prod_written", "prod_pfree", "relay_full_o", "prod_full_a"]
for f in sys.argv[1:]:
    tr = np.load(f)["tr"].astype(np.int64)
    t0 = tr[tr > 0].min()
    print("==", f)
    ncta = max(c for c in range(8) if tr[c].max() > 0) + 1
    for c in range(ncta):
        row = []
        for e in range(8):
            x = tr[c, e]
            v = x[x > 0]
            if len(v) < 10: continue
            d = np.diff(v)
            row.append(f"{EV[e]}: n={len(v)} per={np.median(d):.0f}")
        print(f" cta{c}: " + "; ".join(row))
    # lags on cta 0 (leader), stages 100..600
    i = np.arange(100, 600)
    def lag(a, ca, b, cb, shift=0):
        x = tr[ca, a, i] ; y = tr[cb, b, i - shift]
        ok = (x > 0) & (y > 0)
        return np.median((x - y)[ok]) if ok.any() else float('nan')
    print("  gen (written-empty_o) per cta:", [lag(4, c, 3, c) for c in range(ncta)])
    print("  pfree wait (pfree-written):", [lag(5, c, 4, c) for c in range(ncta)])
    print("  prod full_a - empty_o:", [lag(7, c, 3, c) for c in range(ncta)])
    print("  mma full_o - full_a (leader):", lag(2, 0, 1, 0))
    print("  mma full_o - max(written) lead:", np.median([tr[0, 2, k] - max(tr[c, 4, k] for c in range(ncta)) for k in i]))
    if ncta > 1: print("  relay(peer) - written(peer):", lag(6, 1, 4, 1), " mma full_o - relay:", lag(2, 0, 6, 1))
    print("  mma full_a - tma empty_a:", lag(1, 0, 0, 0))
    print("  per-stage MMA period:", np.median(np.diff(tr[0, 2, i])))
