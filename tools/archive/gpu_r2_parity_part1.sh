# config-4 full parity, part 1 (reference steps 0 -> 10 + ETRD checkpoint in /tmp)
free -g | head -2; nproc; df -h /tmp | tail -1
timeout 3300 python tools/parity_cfg4_full.py part1 gpurun_out/r02_parity_cfg4_full.jsonl > gpurun_out/r02_parity_part1.log 2>&1; echo "part1 rc=$?"; tail -3 gpurun_out/r02_parity_part1.log; ls -la /tmp/etd_cfg4_* 
