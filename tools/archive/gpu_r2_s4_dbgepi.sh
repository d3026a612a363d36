for d in 0 1 2 3; do
ETD_DBG_EPI=$d ETD_CTA_TRACE=x_back_upd ETD_CTA_TRACE_OUT=gpurun_out/s4_trace_upd$d.bin python tools/ab_stage.py 4 1 x_back_upd "" 2> gpurun_out/s4_dbg.err | cut -c1-200
python tools/cta_trace.py gpurun_out/s4_trace_upd$d.bin | sed -n 2,5p
done
