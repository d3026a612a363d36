# full-size parity of the level-2 default path: configs 0-3 against the reference CPU
# implementation, config 4 against the dense path over all 20 steps
timeout 1500 python tools/parity_configs.py gpurun_out/parity_l2.jsonl 0 1 2 3 > gpurun_out/parity_l2.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/parity_l2.log | cut -c1-300
timeout 900 python tools/fold_vs_dense.py gpurun_out/l2_vs_dense.jsonl 0 1 2 3 4 > gpurun_out/l2_vs_dense.log 2>&1; echo "vs dense rc=$?"; cat gpurun_out/l2_vs_dense.jsonl | cut -c1-300
