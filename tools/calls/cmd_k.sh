# TF32 peak; sanitizer case list plain, then under compute-sanitizer memcheck
timeout 120 python tools/measure_tf32_peak.py > gpurun_out/r2k_tf32.log 2>&1
timeout 600 python tools/sanitize_cases.py > gpurun_out/r2k_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2k_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2k_memcheck.log
