for st in z_back_a x_back_src; do
ETD_CTA_TRACE=$st ETD_CTA_TRACE_OUT=gpurun_out/s4_trace_$st.bin python tools/one_step.py 4 > /dev/null 2> gpurun_out/s4_trace.err; echo rc=$?
python tools/cta_trace.py gpurun_out/s4_trace_$st.bin
done
