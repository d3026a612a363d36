# session 4: ncu --set full of the level-2 stack passes (config 3: replay works) + the full-size anchors test
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/s4_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/s4_fullsize.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"etd_source|etd_fold2" -c 3 -o gpurun_out/s4_stack python tools/one_step.py 3 > /dev/null 2>&1; echo "ncu stack rc=$?"
