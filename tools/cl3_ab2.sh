# A/B: clusters of 3 pairs (cta_group=6) vs 4 pairs (8) for the fast transform at several shapes
for N in 50000 25000; do
echo "N=$N"
N=$N CFGS='[["bf16","fast",0,{"CG":6}],["bf16","fast",0,{"CG":8}],["tf32","fast",0,{"CG":6}],["tf32","fast",0,{"CG":8}],["bf16","accurate",0,{"CG":8}]]' ROUNDS=5 timeout 600 python tools/abmulti.py new 2>&1 | tail -5
done
