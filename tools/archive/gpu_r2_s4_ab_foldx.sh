python tools/ab_stage.py 4 3 source,fold_ "ETD_FOLDX4=0" "" > gpurun_out/s4_ab_foldx.jsonl 2> gpurun_out/s4_ab_foldx.err; echo rc=$?; cat gpurun_out/s4_ab_foldx.jsonl; tail -3 gpurun_out/s4_ab_foldx.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_pytest_gpu2.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/s4_pytest_gpu2.log
