#!/usr/bin/env bash
# End-of-round evidence (one gpurun call): tests, smoke, bench lines (C3, C5,
# reference arm), per-config numbers, C4 loop, ncu launch list + full
# captures, sanitizers.  Outputs in gpurun_out/, copied to profiles/ by hand.
set -u
T=${TAG:-r2final}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_${T}.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${T}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${T}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${T}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${T}.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${T}.json 2>&1
timeout 900 python bench.py --config c5_multicorner --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5_${T}.json 2> gpurun_out/bench_c5_${T}.err
timeout 1200 python scripts/bench_configs.py > gpurun_out/bench_configs_${T}.json 2> gpurun_out/bench_configs_${T}.err
timeout 900 python scripts/bench_tdp.py --iters 1000 --check > gpurun_out/bench_c4_${T}.json 2> gpurun_out/bench_c4_${T}.err
# rows f1 / f2: Arnoldi net model (C2 / C4 / C3), Steiner RC (C4 with full parity, C3), latency probe
for cfg in c2_tau c4_tdp c3_superblue; do
timeout 600 python bench.py --config $cfg --net-model arnoldi --steps 10 --warmup 3 --no-cpu-baseline --quick --phases > gpurun_out/bench_arnoldi_${cfg}_${T}.json 2> gpurun_out/bench_arnoldi_${cfg}_${T}.err
done
for cfg in c2_tau c3_superblue; do
timeout 600 python bench.py --config $cfg --exceptions --steps 10 --warmup 3 --no-cpu-baseline --quick > gpurun_out/bench_exc_${cfg}_${T}.json 2> gpurun_out/bench_exc_${cfg}_${T}.err
timeout 600 python bench.py --config $cfg --through --steps 5 --warmup 3 --no-cpu-baseline --quick > gpurun_out/bench_thr_${cfg}_${T}.json 2> gpurun_out/bench_thr_${cfg}_${T}.err
done
timeout 300 python scripts/load_time.py c3_superblue > gpurun_out/load_time_${T}.txt 2>&1
timeout 600 python bench.py --case --steps 10 --warmup 3 --no-cpu-baseline --quick > gpurun_out/bench_case_c3_superblue_${T}.json 2> gpurun_out/bench_case_${T}.err
timeout 300 python scripts/path_time.py c3_superblue > gpurun_out/path_time_c3_${T}.txt 2>&1
timeout 900 python scripts/bench_steiner.py c4_tdp --full-parity > gpurun_out/steiner_c4_${T}.json 2> gpurun_out/steiner_c4_${T}.err
timeout 900 python scripts/bench_steiner.py c3_superblue --reps 3 > gpurun_out/steiner_c3_${T}.json 2> gpurun_out/steiner_c3_${T}.err
timeout 600 python scripts/latency_probe.py > gpurun_out/latency_${T}.txt 2>&1
# functional multi-rank check on the one GPU (gloo): C5 as 2 ranks x 4 corners
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --dist-backend gloo --steps 10 --warmup 3 --quick 2> gpurun_out/multirank_${T}.err | tail -1 > gpurun_out/multirank_${T}.json
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${T}.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch_${T}.log 2>&1
for K in fwd_persistent bwd_persistent rc_warp tc_event tc_node tc_w; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip 3 --launch-count 1 -o gpurun_out/prof_${T}_${K} \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_${T}.log 2>&1
done
fi
# compute-sanitizer is closed on the GPU pool since r2final2 (rc 86); opt in with SAN=1
if [ "${SAN:-0}" = 1 ]; then
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_${tool}_${T}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_${tool}_${T}.log
done
fi
