python tools/quick_perf.py 0 1 2 3 --steps 5 > gpurun_out/s4_quick_perf.jsonl 2> gpurun_out/s4_quick_perf.err; echo rc=$?
