mkdir -p gpurun_out
for d in 0 1 2; do python tools/run_layer.py --layer conv4_2a --dir $d --time | head -1; done
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair|conv_tc_kernel|conv_tma_wgrad" -s 1 -c 1 -o gpurun_out/c4_2a_fwd python tools/run_layer.py --layer conv4_2a --dir 0 --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair|conv_tc_kernel|conv_tma_wgrad" -s 1 -c 1 -o gpurun_out/c4_2a_dgrad python tools/run_layer.py --layer conv4_2a --dir 1 --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_pair|conv_tc_kernel|conv_tma_wgrad" -s 1 -c 1 -o gpurun_out/c4_2a_wgrad python tools/run_layer.py --layer conv4_2a --dir 2 --iters 2 > /dev/null 2>&1
ls -la gpurun_out
