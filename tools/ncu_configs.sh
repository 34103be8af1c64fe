set -x
for cfg in c2 c3 c4; do
  for prec in mixed fp64; do
    timeout 300 python bench.py --config $cfg --precision $prec --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/pre_${cfg}_${prec}.log 2>&1 || continue
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep_ -c 16 --csv --log-file gpurun_out/launches_${cfg}_${prec}.csv python bench.py --config $cfg --precision $prec --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/ncu_${cfg}_${prec}.log 2>&1
  done
done
