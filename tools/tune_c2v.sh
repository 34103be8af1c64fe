# C2 v-sweep (strided, outer) knob matrix: stages (SLDG_TMA_SDIV), CTAs per SM, tile width
mkdir -p gpurun_out/c2v
for cfg in "2 1 64" "3 1 64" "4 1 64" "6 1 64" "2 2 64" "4 2 64" "4 1 32" "4 1 128"; do
  set -- $cfg
  SLDG_TMA_SDIV=$1 SLDG_TMA_CTAS=$2 SLDG_TMA_W=$3 timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/c2v/s$1_c$2_w$3.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/c2v/s$1_c$2_w$3.log').read().strip().splitlines()[-1]); print('sdiv=$1 ctas=$2 W=$3', round(d['value'],1), {k: round(v['ms_per_launch']*1e3,1) for k, v in d['sweeps'].items()})"
done
