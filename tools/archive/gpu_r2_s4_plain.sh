python tools/ab_stage.py 4 3 z_back_a,y_back_a,x_back_src,x_back_upd,x_fwd_corr "" 2> gpurun_out/s4_plain.err | cut -c1-400
