# same-box A/B of whole cfg4 steps across library builds: bash scripts/cfg4_lib_ab.sh libA.so libB.so ...
for r in 1 2; do
  for lib in "$@"; do
    EDL_LIB=$lib timeout 300 python -c "
import os,sys; sys.argv=['x']; sys.path.insert(0,'scripts'); import cfg4_student_bench as c
s=c.run(256); t=c.run(256, with_teacher=True)
print(os.environ['EDL_LIB'], 'student', s['samples_per_s'], s['ms'], 'online', t['samples_per_s'], t['ms'], flush=True)
" >> gpurun_out/cfg4_lib_ab.txt 2>&1
  done
done
