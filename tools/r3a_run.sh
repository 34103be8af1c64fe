O=gpurun_out/r3a; mkdir -p $O
bash tools/env_sweep.sh SLDG_KEEP_OVERLAP "1 0 1 0" c5 c4 > $O/keep_env.txt 2>&1
bash tools/ab_run.sh _ab_head head . keep c5 c5 c3 > $O/keep_vs_head.txt 2>&1
