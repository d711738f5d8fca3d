#!/bin/bash
# Round-end measurement pass on the GPU box: everything lands in gpurun_out/ (copied to profiles/ afterwards).
set -x
python scripts/bench_configs.py > gpurun_out/configs.log 2>&1
python scripts/parity_report.py > gpurun_out/parity.log 2>&1
python scripts/precision_check.py --full > gpurun_out/precision_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:march_mma -s 3 -c 1 -o gpurun_out/ncu_filter_final -f python scripts/prof_frame.py 1 > gpurun_out/ncu1.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_filter_final.ncu-rep > gpurun_out/ncu_r1_filter_v3.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_filter_final.ncu-rep 16 >> gpurun_out/ncu_r1_filter_v3.summary.txt
ncu --set full --clock-control none --import-source on -k regex:march_small -s 6 -c 1 -o gpurun_out/ncu_exact_final -f python scripts/prof_frame.py 1 > gpurun_out/ncu2.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_exact_final.ncu-rep > gpurun_out/ncu_r1_exact_v7.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_exact_final.ncu-rep 16 >> gpurun_out/ncu_r1_exact_v7.summary.txt
BENCH_PREHEAT=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r1_v10.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log > gpurun_out/bench_r1_v10.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_march.py -q -k "decision_filter or distilled_matches" > gpurun_out/sanitizer_memcheck.log 2>&1
tail -3 gpurun_out/*.log | cut -c1-300
