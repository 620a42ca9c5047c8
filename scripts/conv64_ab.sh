# same-box A/B of the 64-channel 3x3 conv paths: EDL_LIB=<lib> variants, interleaved
for r in 1 2 3; do
  for lib in "$@"; do
    echo -n "$lib " >> gpurun_out/conv64_ab.txt
    EDL_LIB=$lib python scripts/conv64_bench.py >> gpurun_out/conv64_ab.txt 2>&1
  done
  echo -n "im2col " >> gpurun_out/conv64_ab.txt
  EDL_HALO=0 python scripts/conv64_bench.py >> gpurun_out/conv64_ab.txt 2>&1
done
