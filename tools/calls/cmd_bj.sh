# the GPU suite against the SK_DEBUG_HANG build (every mbarrier wait bounded; a stuck wait traps with
# its barrier / parity / CTA) -- the box works on a copy of the repo, so the debug .so replaces the
# in-tree one there only
cp ab_old/debughang/libsketch.so paper_2603_20966_b200/libsketch.so
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2bj_tests.log 2>&1
tail -3 gpurun_out/r2bj_tests.log
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2bj_cases.log 2>&1
tail -2 gpurun_out/r2bj_cases.log
