# end-of-round config-4 full parity, part 1 (reference steps 0 -> 10 + ETRD checkpoint in /tmp)
free -g | head -2; nproc
ETD_PARITY_SCHEDULES=default timeout 3300 python tools/parity_cfg4_full.py part1 gpurun_out/r02_parity_cfg4_full_end.jsonl > gpurun_out/s4_parity_part1.log 2>&1; echo "part1 rc=$?"; tail -2 gpurun_out/s4_parity_part1.log | cut -c1-400; ls -la /tmp/etd_cfg4_*
