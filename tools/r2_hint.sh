# mbarrier wait: suspend-time hint A/B at C5 (forced variant builds on the box)
O=gpurun_out/hint; mkdir -p $O
B="--no-cpu-baseline --no-compare-fp64 --no-vlasov"
run() { for i in 1 2; do timeout 300 python bench.py $B > $O/$1_$i.json 2>/dev/null; done; }
run def
for h in 0 20000; do SLDG_NVCC_EXTRA="-DSLDG_MBAR_HINT_NS=${h}u" python -m paper_1603_07008_b200._build --force > $O/build_$h.log 2>&1; run h$h; done
