# pipeline traces (trace-enabled build in ab_old/trace): c4 shape (single pass, 16-CTA clusters) and c2
timeout 600 python tools/trace4.py '[["bf16","fast",0,0,2048,1000000,512],["bf16","fast",0,0,50000,50000,256]]' > gpurun_out/r2t_trace.log 2>&1
