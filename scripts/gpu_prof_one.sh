set -u
mkdir -p gpurun_out
T=${T:-x}; K=${K:-fwd_persistent}
python -m paper_2511_11660_b200.build --force > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip 3 --launch-count 1 -o gpurun_out/prof_${T}_${K} \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_${T}.log 2>&1
