for h in 1 0 1 0; do
EDL_HALO=$h timeout 300 python -c "
import os,sys; sys.argv=['x']; sys.path.insert(0,'scripts'); import cfg4_student_bench as c
print('halo', os.environ['EDL_HALO'], c.run(256), c.run(256, with_teacher=True), flush=True)
" >> gpurun_out/cfg4_halo_ab.txt 2>&1
done
CFG4_PROFILE=1 CFG4_BATCH=256 CFG4_TEACHER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg4_halo_launches.csv python scripts/cfg4_student_bench.py > gpurun_out/cfg4_halo_ncu.log 2>&1
