#!/bin/bash
# Round-end measurement pass on the GPU box: everything lands in gpurun_out/ (copied to profiles/ afterwards).
python -m pytest tests -m gpu -q -s > gpurun_out/gpu_tests_final.log 2>&1; tail -3 gpurun_out/gpu_tests_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err
BENCH_PREHEAT=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python scripts/launch_list.py gpurun_out/launches_final.csv > gpurun_out/launches_final.summary.txt
ncu --set full --clock-control none --import-source on -k regex:march_tc5 -s 2 -c 1 -o gpurun_out/ncu_final_tc5 -f python scripts/prof_frame.py 2 > gpurun_out/ncu1.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_final_tc5.ncu-rep > gpurun_out/ncu_final_tc5_filter.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_final_tc5.ncu-rep 16 >> gpurun_out/ncu_final_tc5_filter.summary.txt
ncu --set full --clock-control none --import-source on -k regex:march_tail -s 1 -c 1 -o gpurun_out/ncu_final_tail -f python scripts/prof_frame.py 2 > gpurun_out/ncu2.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_final_tail.ncu-rep > gpurun_out/ncu_final_tail.summary.txt; python scripts/ncu_opcodes.py gpurun_out/ncu_final_tail.ncu-rep 12 >> gpurun_out/ncu_final_tail.summary.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
tail -c 400 gpurun_out/bench_final.json; tail -c 600 gpurun_out/bench_reference_final.json; head -12 gpurun_out/launches_final.summary.txt
