# pipeline trace of the final c2 kernel (8 bf16 producer warps)
timeout 600 python tools/trace4.py '[["bf16","fast",0,0,50000,50000,256]]' > gpurun_out/r2an_trace.log 2>&1
