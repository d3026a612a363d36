# end-of-round config-4 full parity, part 2 (reference steps 10 -> 20 from part 1's /tmp ETRD checkpoint)
ls -la /tmp/etd_cfg4_* || echo "NO CHECKPOINT (different box)"
ETD_PARITY_SCHEDULES=default,dense timeout 3300 python tools/parity_cfg4_full.py part2 gpurun_out/r02_parity_cfg4_full_end.jsonl > gpurun_out/s4_parity_part2.log 2>&1; echo "part2 rc=$?"; tail -3 gpurun_out/s4_parity_part2.log | cut -c1-400
