# Late round-2 evidence: launch list + DRAM bytes of C3 fp64 (windowed d = 0 kernel), and a full
# capture of sweep_d0_win.  -> gpurun_out/ev3/
set -x
O=gpurun_out/ev3
mkdir -p $O
cp profiles/ncu_dram.json $O/ncu_dram.json
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov --no-graph"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep_ -c 16 --csv"
timeout 600 python bench.py --steps 1 --warmup 3 $B --config c3 --precision fp64 > $O/pre_c3_fp64.log 2>&1
timeout 1200 ncu $M --log-file $O/launches_c3_fp64.csv python bench.py --steps 1 --warmup 3 $B --config c3 --precision fp64 > $O/ncu_c3_fp64.log 2>&1
python tools/ncu_summary.py launches $O/launches_c3_fp64.csv $O/launches_c3_fp64.md --dram-json $O/ncu_dram.json --key c3_fp64_k4_D2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_d0_win -s 3 -c 1 -o $O/full_d0win_c3 python bench.py --steps 1 --warmup 3 $B --config c3 --precision fp64 > $O/ncu_full_d0win.log 2>&1
python tools/ncu_summary.py full $O/full_d0win_c3.ncu-rep $O/ncu_full_d0win_c3.md
rm -f $O/*.ncu-rep
