#!/bin/bash
# Same build, one environment variable swept: env_sweep.sh VAR "v1 v2 ..." config... (bench.py, kernel-only)
mkdir -p gpurun_out/envsweep
VAR=$1; VALS=$2; shift 2
for c in "$@"; do
  for v in $VALS; do
    env $VAR=$v timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/envsweep/${VAR}_${v}_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/envsweep/${VAR}_${v}_$c.log').read().strip().splitlines()[-1]); print('$VAR=$v $c', round(d['value'],1), {k: round(v['ms_per_launch']*1e3,1) for k, v in d['sweeps'].items()}, d['clocks']['sm_mhz'])"
  done
done
