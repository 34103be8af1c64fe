# Round-2 final evidence: GPU tests, smoke, the default bench line (with its reference arm), bench
# lines of the other configs / precisions, and the unfused C5 split step.  -> gpurun_out/final/
O=${O:-gpurun_out/final}; mkdir -p $O
nvidia-smi -q -d CLOCK,POWER > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
B="--no-cpu-baseline --no-vlasov"
for c in c4 c3 c2; do
  timeout 300 python bench.py --config $c $B > $O/bench_$c.json 2> $O/bench_$c.err
  timeout 300 python bench.py --config $c --precision fp64 $B --no-compare-fp64 > $O/bench_${c}_fp64.json 2> $O/bench_${c}_fp64.err
done
timeout 300 python bench.py --no-fuse-x $B > $O/bench_c5_unfused.json 2> $O/bench_c5_unfused.err
timeout 300 python bench.py --eps 0.5 $B --no-compare-fp64 > $O/bench_c5_eps05.json 2> $O/bench_c5_eps05.err
