python tools/solo_rank.py 4 1 8 4 2 > gpurun_out/s4_solo_rank_cfg4.jsonl 2> gpurun_out/s4_solo.err; echo rc=$?; cat gpurun_out/s4_solo_rank_cfg4.jsonl; tail -3 gpurun_out/s4_solo.err
