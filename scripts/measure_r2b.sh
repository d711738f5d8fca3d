#!/bin/bash
# Measurement pass after the refined Lipschitz bounds (everything lands in gpurun_out/).
python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
BENCH_PREHEAT=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python scripts/launch_list.py gpurun_out/launches_r2b.csv > gpurun_out/launches_r2b.summary.txt
ncu --set full --clock-control none --import-source on -k regex:march_tc5 -s 12 -c 1 -o gpurun_out/ncu_r2b_tc5 -f python scripts/prof_frame.py 2 > gpurun_out/ncu1.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_r2b_tc5.ncu-rep > gpurun_out/ncu_r2b_tc5_filter.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_r2b_tc5.ncu-rep 16 >> gpurun_out/ncu_r2b_tc5_filter.summary.txt
ncu --set full --clock-control none --import-source on -k regex:march_small -s 18 -c 1 -o gpurun_out/ncu_r2b_small -f python scripts/prof_frame.py 2 > gpurun_out/ncu2.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_r2b_small.ncu-rep > gpurun_out/ncu_r2b_exact_small.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_r2b_small.ncu-rep 16 >> gpurun_out/ncu_r2b_exact_small.summary.txt
ncu --set full --clock-control none --import-source on -k regex:lip_bound -c 1 -o gpurun_out/ncu_r2b_lip -f python scripts/prof_frame.py 1 > gpurun_out/ncu3.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_r2b_lip.ncu-rep > gpurun_out/ncu_r2b_lip_bound.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_r2b_lip.ncu-rep 16 >> gpurun_out/ncu_r2b_lip_bound.summary.txt
tail -c 600 gpurun_out/bench_r2b.json; cat gpurun_out/launches_r2b.summary.txt | head -24
