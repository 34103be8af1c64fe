O=gpurun_out/vnk4; mkdir -p $O
B="--no-cpu-baseline --no-compare-fp64"
run() { for i in 1 2; do timeout 300 python bench.py --config c3 $B > $O/$1_$i.json 2>/dev/null; done; }
run m3
for mb in 2 1; do SLDG_NVCC_EXTRA="-DSLDG_VN_K4_MINB=$mb" python -m paper_1603_07008_b200._build --force > $O/build_$mb.log 2>&1; run m$mb; done
