# Round-2 evidence on one GPU (run under gpurun): ncu launch lists with DRAM bytes per launch for
# the bench configs (default = fused x pair; C5 also unfused), full-set captures of the fused pair
# and of a strided v sweep at C5 size.  Outputs under gpurun_out/ev2/ (copied into profiles/round2).
set -x
O=gpurun_out/ev2
mkdir -p $O
cp profiles/ncu_dram.json $O/ncu_dram.json
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov --no-graph"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep_ -c 16 --csv"
run() {  # run <tag> <key> <bench args...>
  tag=$1; key=$2; shift 2
  timeout 600 python bench.py --steps 1 --warmup 3 $B "$@" > $O/pre_$tag.log 2>&1 || return
  timeout 1200 ncu $M --log-file $O/launches_$tag.csv python bench.py --steps 1 --warmup 3 $B "$@" > $O/ncu_$tag.log 2>&1
  python tools/ncu_summary.py launches $O/launches_$tag.csv $O/launches_$tag.md --dram-json $O/ncu_dram.json --key $key
}
run c5_mixed c5_mixed_k3_D4 --config c5
run c5_mixed_nofuse c5_mixed_k3_D4 --config c5 --no-fuse-x
run c4_mixed c4_mixed_k2_D4 --config c4
run c4_fp64 c4_fp64_k2_D4 --config c4 --precision fp64
run c3_mixed c3_mixed_k4_D2 --config c3
run c3_fp64 c3_fp64_k4_D2 --config c3 --precision fp64
run c2_mixed c2_mixed_k4_D2 --config c2
run c2_fp64 c2_fp64_k4_D2 --config c2 --precision fp64
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/full_fused_c5 python bench.py --steps 1 --warmup 3 $B > $O/ncu_full_fused.log 2>&1
python tools/ncu_summary.py full $O/full_fused_c5.ncu-rep $O/ncu_full_fused_c5.md
python tools/ncu_hotloop.py $O/full_fused_c5.ncu-rep 30 > $O/ncu_hotloop_fused_c5.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_strided -s 6 -c 1 -o $O/full_strided_c5 python bench.py --steps 1 --warmup 3 $B > $O/ncu_full_strided.log 2>&1
python tools/ncu_summary.py full $O/full_strided_c5.ncu-rep $O/ncu_full_strided_c5.md
python tools/ncu_hotloop.py $O/full_strided_c5.ncu-rep 30 > $O/ncu_hotloop_strided_c5.txt
rm -f $O/*.ncu-rep
