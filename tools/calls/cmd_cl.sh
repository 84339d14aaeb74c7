# c2: idle-SM side launch potential (second stream, unshared pairs)
timeout 600 python tools/side_ab.py > gpurun_out/r2cl_side.txt 2>&1
SIDE_CG=1 SIDES=128,256,512 timeout 600 python tools/side_ab.py >> gpurun_out/r2cl_side.txt 2>&1
