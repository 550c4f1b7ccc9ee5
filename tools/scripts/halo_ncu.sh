ncu --set full --clock-control none --import-source on -k regex:"conv_halo" -s 1 -c 1 -o gpurun_out/halo_c22b_fwd python tools/run_layer.py --layer conv2_2b --dir 0 --iters 2 > /dev/null 2>&1
PK_HALO_TRACE=1 timeout 60 python tools/run_layer.py --layer conv2_2b --dir 0 --iters 2 2>&1 | tail -32 > gpurun_out/halo_trace.txt
