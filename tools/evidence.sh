# Round evidence refresh on one GPU (run under gpurun): GPU tests, ncu launch lists with DRAM
# bytes per sweep (C2-C4 mixed + fp64, C5 mixed), a full-set capture of C2's strided sweep.
# Outputs under gpurun_out/ev3/ (copied into profiles/ by hand).
set -x
O=gpurun_out/ev3
mkdir -p $O
cp profiles/ncu_dram.json $O/ncu_dram.json
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
B="--no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov --no-graph"
for cfg in c2 c3 c4; do
  for prec in mixed fp64; do
    timeout 300 python bench.py --config $cfg --precision $prec --steps 1 --warmup 3 $B > $O/pre_${cfg}_${prec}.log 2>&1 || continue
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep_ -c 16 --csv --log-file $O/launches_${cfg}_${prec}.csv python bench.py --config $cfg --precision $prec --steps 1 --warmup 3 $B > $O/ncu_${cfg}_${prec}.log 2>&1
    k=$(python -c "import bench; print(bench.CONFIGS['$cfg'][2])")
    D=$(python -c "import bench; print(len(bench.CONFIGS['$cfg'][0]))")
    python tools/ncu_summary.py launches $O/launches_${cfg}_${prec}.csv $O/launches_${cfg}_${prec}.md --dram-json $O/ncu_dram.json --key ${cfg}_${prec}_k${k}_D${D}
  done
done
timeout 600 python bench.py --steps 1 --warmup 3 $B > $O/pre_c5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep_ -c 16 --csv --log-file $O/launches_c5_mixed.csv python bench.py --steps 1 --warmup 3 $B > $O/ncu_c5.log 2>&1
python tools/ncu_summary.py launches $O/launches_c5_mixed.csv $O/launches_c5_mixed.md --dram-json $O/ncu_dram.json --key c5_mixed_k3_D4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_strided -s 3 -c 1 -o /tmp/c2s python bench.py --config c2 --steps 1 --warmup 3 $B > $O/ncu_full_c2s.log 2>&1
python tools/ncu_summary.py full /tmp/c2s.ncu-rep $O/ncu_full_c2s.md
