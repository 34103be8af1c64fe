for t in 24 32 40 48; do SLDG_TMA_TSUB=$t timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t2_$t.log 2>&1; done
for t in 32 48 64; do SLDG_TMA_TSUB=$t timeout 300 python bench.py --config c2 --precision fp64 --no-cpu-baseline --no-e2e --no-compare-fp64 --no-vlasov > gpurun_out/t2f_$t.log 2>&1; done
