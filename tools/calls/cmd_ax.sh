# tf32 cluster sizes (accurate / fast transform)
CFGS='[["tf32","accurate",0],["tf32","accurate",0,{"CG":6}],["tf32","accurate",0,{"CG":4}],["tf32","fast",0],["tf32","fast",0,{"CG":6}]]' ROUNDS=3 timeout 900 python tools/abmulti.py new > gpurun_out/r2ax.txt 2>&1
