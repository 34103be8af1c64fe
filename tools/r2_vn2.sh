O=gpurun_out/vn2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vnodes.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnode_sweep_multi -s 2 -c 1 -o $O/full_vn_multi_c5s python tools/diag_vnodes.py c5s > $O/ncu_multi.log 2>&1
SLDG_VN_MULTI=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:vnode_sweep_kernel -s 2 -c 1 -o $O/full_vn_one_c5s python tools/diag_vnodes.py c5s > $O/ncu_one.log 2>&1
