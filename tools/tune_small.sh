for c in c2 c3 c4; do
 for w in 256 128 64; do
  for t in 64 16 8; do
   SLDG_TMA_W=$w SLDG_TMA_TSUB=$t timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t_${c}_${w}_${t}.log 2>&1
  done
 done
done
