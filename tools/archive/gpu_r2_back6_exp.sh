# back6 MODE 0 nondeterminism experiments
S=x_back_src,x_back_upd
timeout 120 python tools/back6_repeat.py 255 $S
ETD_FORCE_TILE=0 timeout 120 python tools/back6_repeat.py 255 $S
ETD_FORCE_TILE=2 timeout 120 python tools/back6_repeat.py 255 $S
ETD_FORCE_TILE=0 timeout 120 python tools/back6_repeat.py 255 z_back_a,y_back_a
timeout 120 python tools/back6_repeat.py 127 $S
ETD_BACK6=0 timeout 120 python tools/back6_repeat.py 255 x_back_src_o,x_back_src_e
ETD_BACK6=0 timeout 300 python tools/check_cfg4_sample.py gpurun_out/r02_cfg4_sample_checks.jsonl r01_unfold
