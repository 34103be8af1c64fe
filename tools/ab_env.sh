# A/B of an environment setting on the same build: ab_env.sh "<envA>" "<envB>" <configs...>
mkdir -p gpurun_out/ab
A=$1; B=$2; shift 2
run() {  # run <env> <tag> <config>
  env $1 timeout 400 python bench.py --config $3 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/ab/$2_$3.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab/$2_$3.log').read().strip().splitlines()[-1]); print('$2 $3', round(d['value'],1), {k: round(v['ms_per_launch']*1e3,1) for k, v in d['sweeps'].items()}, d['clocks']['sm_mhz'])"
}
for c in "$@"; do run "$A" A $c; run "$B" B $c; done
