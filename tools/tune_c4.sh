for ctas in 2 1; do
 for dd in 2 3 4 6; do
  SLDG_TMA_CTAS=$ctas SLDG_TMA_D0DIV=$dd timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t4_${ctas}_${dd}.log 2>&1
 done
done
