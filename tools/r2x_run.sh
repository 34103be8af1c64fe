O=gpurun_out/r2x; mkdir -p $O
timeout 600 python tools/order_sweep.py --reps 5 --out $O/order_base.md > $O/base.log 2>&1
(cd _ab_split && timeout 600 python tools/order_sweep.py --reps 5 --out $GRAFT_REPO_ROOT/$O/order_split.md > $GRAFT_REPO_ROOT/$O/split.log 2>&1)
(cd _ab_split && timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "high_order or randomized or single_sweeps" > $GRAFT_REPO_ROOT/$O/pytest_split.log 2>&1; echo rc=$? >> $GRAFT_REPO_ROOT/$O/pytest_split.log)
