for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/probes/sanitizer_halo.py > gpurun_out/r02_san_${tool}_halo.txt 2>&1; echo "$tool rc=$?" >> gpurun_out/r02_san_${tool}_halo.txt
done
PK_HALO_PAIR=1 timeout 900 compute-sanitizer --tool memcheck python tools/probes/sanitizer_halo.py > gpurun_out/r02_san_memcheck_halo_pair.txt 2>&1; echo "rc=$?" >> gpurun_out/r02_san_memcheck_halo_pair.txt
