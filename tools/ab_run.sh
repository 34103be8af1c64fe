# A/B of two built trees on the same box: ab_run.sh <dirA> <nameA> <dirB> <nameB> <configs...>
mkdir -p gpurun_out/ab
run() {  # run <dir> <name> <config>
  (cd $1 && timeout 400 python bench.py --config $3 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > $GRAFT_REPO_ROOT/gpurun_out/ab/$2_$3.log 2>&1)
  python -c "import json; d=json.loads(open('gpurun_out/ab/$2_$3.log').read().strip().splitlines()[-1]); print('$2 $3', round(d['value'],1), {k: round(v['ms_per_launch']*1e3,1) for k, v in d['sweeps'].items()}, d['clocks']['sm_mhz'])"
}
A=$1; NA=$2; B=$3; NB=$4; shift 4
for c in "$@"; do run $A $NA $c; run $B $NB $c; done
