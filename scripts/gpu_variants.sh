#!/usr/bin/env bash
# Tuning sweep in one gpurun call: each variant is libsta built with extra nvcc
# flags into gpurun_out/var/, then timed by bench.py (STA_LIB_PATH selects it).
#   TAG=r2d VARIANTS="base:;nopf:-DSTA_FWD_PF=0" CFGS="c3_superblue c5_multicorner" scripts/gpu_variants.sh
set -u
TAG=${TAG:-var}
mkdir -p gpurun_out/var
IFS=';' read -ra VS <<< "${VARIANTS:-base:}"
for v in "${VS[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  python -m paper_2511_11660_b200.build --out gpurun_out/var/libsta_${name}.so --flags="$flags" > gpurun_out/var/build_${name}.log 2>&1 &
done
wait
for rep in 1 2; do
for v in "${VS[@]}"; do
  name=${v%%:*}
  for cfg in ${CFGS:-c3_superblue}; do
    STA_LIB_PATH=gpurun_out/var/libsta_${name}.so timeout 600 python bench.py --config $cfg --quick --phases --steps ${STEPS:-30} \
      > gpurun_out/var/${TAG}_${name}_${cfg}_${rep}.json 2> gpurun_out/var/${TAG}_${name}_${cfg}_${rep}.err
    python - "$name" "$cfg" "gpurun_out/var/${TAG}_${name}_${cfg}_${rep}.json" <<'PY' >> gpurun_out/var/${TAG}_summary.txt
import json, sys
try:
    j = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    ph = j.get("phases_ms", {})
    print(f"{sys.argv[1]:12s} {sys.argv[2]:16s} ms={j['ms_per_step']:.4f} rc={ph.get('rc', 0):.4f} "
          f"fwd={ph.get('forward', 0):.4f} bwd={ph.get('backward', 0):.4f} clocks={j.get('clocks', {}).get('sm_mhz')}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done
done
cat gpurun_out/var/${TAG}_summary.txt
