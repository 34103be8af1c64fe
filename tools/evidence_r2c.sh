# Late round-2 launch lists of every bench config with DRAM bytes AND the secondary roofline
# (fp64 pipe, XU) per launch -> gpurun_out/ev4/ (ncu_dram.json, ncu_pipe.json, launches_*.md)
set -x
O=gpurun_out/ev4
mkdir -p $O
cp profiles/ncu_dram.json $O/ncu_dram.json
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov --no-graph"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k regex:sweep_ -c 16 --csv"
run() {  # run <tag> <key> <bench args...>
  tag=$1; key=$2; shift 2
  timeout 600 python bench.py --steps 1 --warmup 3 $B "$@" > $O/pre_$tag.log 2>&1 || return
  timeout 1200 ncu $M --log-file $O/launches_$tag.csv python bench.py --steps 1 --warmup 3 $B "$@" > $O/ncu_$tag.log 2>&1
  python tools/ncu_summary.py launches $O/launches_$tag.csv $O/launches_$tag.md --dram-json $O/ncu_dram.json --pipe-json $O/ncu_pipe.json --key $key
}
run c5_mixed c5_mixed_k3_D4 --config c5
run c4_mixed c4_mixed_k2_D4 --config c4
run c4_fp64 c4_fp64_k2_D4 --config c4 --precision fp64
run c3_mixed c3_mixed_k4_D2 --config c3
run c3_fp64 c3_fp64_k4_D2 --config c3 --precision fp64
run c2_mixed c2_mixed_k4_D2 --config c2
run c2_fp64 c2_fp64_k4_D2 --config c2 --precision fp64
