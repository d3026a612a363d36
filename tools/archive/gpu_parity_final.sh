# full-size parity of the final schedule: configs 0-3 vs the reference CPU implementation,
# configs 1-4 vs the dense path (config 4 over all 20 steps)
timeout 900 python tools/fold_vs_dense.py gpurun_out/vs_dense_final.jsonl 1 2 3 4 > gpurun_out/vs_dense_final.log 2>&1; echo "vs dense rc=$?"; cut -c1-220 gpurun_out/vs_dense_final.jsonl
timeout 1800 python tools/parity_configs.py gpurun_out/parity_final.jsonl 0 1 2 3 > gpurun_out/parity_final.log 2>&1; echo "parity rc=$?"; cut -c1-220 gpurun_out/parity_final.jsonl
