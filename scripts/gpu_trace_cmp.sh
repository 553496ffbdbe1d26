#!/usr/bin/env bash
# Per-unit STA_TRACE timelines of the current library and a variant
# (STA_LIB_PATH), then one ncu --set full capture of a kernel of the current
# library with its source page.   T=x K=fwd_persistent VAR=tmpvar/libsta_old.so
set -u
mkdir -p gpurun_out
T=${T:-x}; K=${K:-fwd_persistent}
python __graft_entry__.py > /dev/null 2>&1
timeout 600 python scripts/trace_run.py c3_superblue gpurun_out/trace_${T}_cur.csv > gpurun_out/trace_${T}_cur.txt 2>&1
if [ -n "${VAR:-}" ]; then
STA_LIB_PATH=$VAR timeout 600 python scripts/trace_run.py c3_superblue gpurun_out/trace_${T}_var.csv > gpurun_out/trace_${T}_var.txt 2>&1
fi
rm -f gpurun_out/trace_${T}_*.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip 3 --launch-count 1 -o gpurun_out/prof_${T}_${K} \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_${T}.log 2>&1
ncu -i gpurun_out/prof_${T}_${K}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${T}_${K}.csv 2>/dev/null
ncu -i gpurun_out/prof_${T}_${K}.ncu-rep --page raw --csv > gpurun_out/raw_${T}_${K}.csv 2>/dev/null
