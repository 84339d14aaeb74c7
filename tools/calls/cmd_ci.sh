# sketch time vs Omega row offset k0 for a 25000^2 block
timeout 300 python tools/k0_ab.py > gpurun_out/r2ci_k0.txt 2>&1
