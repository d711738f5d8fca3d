#!/bin/bash
# find the first-wavefront launch of march_tc5_kernel (every first sample of the frame) and capture it with ncu --set full
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:march_tc5 -c 40 --csv --log-file gpurun_out/tc5_list.csv python scripts/prof_frame.py 4 > /dev/null 2>&1
IDX=$(python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/tc5_list.csv')))
for i,r in enumerate(rows):
    if r and r[0]=='ID': h=r; start=i+1; break
vi=h.index('Metric Value')
d=[float(r[vi].replace(',','')) for r in rows[start:] if len(r)>vi]
# the w0 launches are the longest ones; take the last of them
m=max(d); idx=[i for i,v in enumerate(d) if v>0.8*m]
print(idx[-1])
PY
)
echo "w0 launch index $IDX"
ncu --set full --clock-control none --import-source on -k regex:march_tc5 -s $IDX -c 1 -o gpurun_out/ncu_tc5_w0 -f python scripts/prof_frame.py 4 > gpurun_out/ncu1.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_tc5_w0.ncu-rep | head -30
python scripts/ncu_lines.py gpurun_out/ncu_tc5_w0.ncu-rep 24 | tail -26
