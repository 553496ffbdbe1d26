#!/usr/bin/env bash
# Time the current library against variant libraries (STA_LIB_PATH) on C3 / C5.
#   LIBS="old:tmpvar/libsta_old.so new:" CFGS="c3_superblue" scripts/gpu_cmp.sh
set -u
mkdir -p gpurun_out
T=${T:-cmp}
for rep in 1 2; do
for v in ${LIBS:-cur:}; do
  name=${v%%:*}; lib=${v#*:}
  for cfg in ${CFGS:-c3_superblue}; do
    if [ -n "$lib" ]; then export STA_LIB_PATH=$lib; else unset STA_LIB_PATH; fi
    timeout 600 python bench.py --config $cfg --quick --phases --steps ${STEPS:-30} > gpurun_out/${T}_${name}_${cfg}.json 2> gpurun_out/${T}_${name}_${cfg}.err
    python - "$name" "$cfg" "gpurun_out/${T}_${name}_${cfg}.json" <<'PY'
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
