for X in 8 4; do
ETD_XFER_CHUNKS=$X python tools/e2e_timeline.py 2>&1 | grep ETD_TIMELINE > gpurun_out/r2_tl_$X.txt
echo "X=$X $(grep -E ' (up0|col0|col[0-9]+|down[0-9]+) ' gpurun_out/r2_tl_$X.txt | awk '{printf "%s=%s ", $2, $3}')"
done
