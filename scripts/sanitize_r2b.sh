#!/bin/bash
# compute-sanitizer over the kernels added / changed in the second half of round 2 (output: gpurun_out/sanitizer_r2b.txt)
{
echo "== memcheck: Lipschitz refinement + certified skipping (filter, tail) tests"
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_filter.py -q -k "lipschitz or skipping or t_ranges or step_budgets" 2>&1 | tail -6
echo "== racecheck: lip_bound_kernel + march_tc5_kernel + march_tail_kernel on a small march (8^3 field, 96x96 rays)"
KNF_LIP_WIDTH=0.03 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_filter.py -q -k "step_budgets" 2>&1 | tail -6
} > gpurun_out/sanitizer_r2b.txt 2>&1
tail -20 gpurun_out/sanitizer_r2b.txt
