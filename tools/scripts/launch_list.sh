# ncu launch list of one bench step + one full capture of the 64-channel halo kernel
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/run_step.py > gpurun_out/launches_raw.csv 2> gpurun_out/launches_err.txt
ncu --set full --clock-control none --import-source on -k regex:"conv_halo" -s 1 -c 1 -o gpurun_out/r02_halo_mt2_conv2_2b_fwd python tools/run_layer.py --layer conv2_2b --dir 0 --iters 2 > /dev/null 2>&1
ls -la gpurun_out | tail -5
