# which environment does ncu give the profiled process?
ncu --metrics gpu__time_duration.sum python -c "import os; print(sorted((k, v[:80]) for k, v in os.environ.items() if any(t in k for t in (\"INJ\", \"NV\", \"CUDA\", \"PRELOAD\", \"NSIGHT\", \"PROF\"))))" > gpurun_out/r2cv_env.txt 2>&1
