set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
CHEBFD_B200_LIB=$PWD/build/ab/libchebfd_r01.so timeout 600 python tools/band_exp.py --cases c2,c4 --bytes -1 --deg 60
timeout 900 python tools/band_exp.py --cases c4,c3_256,c3_32,c2 --bytes 0,16,32,64 --dyn 0,1 --deg 60
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 600 python tools/prof_case.py --band 16 --dyn 1 && \
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 3 --csv --log-file gpurun_out/ncu_c4_b16_dyn.csv python tools/prof_case.py --band 16 --dyn 1
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 3 --csv --log-file gpurun_out/ncu_c4_b0_dyn.csv python tools/prof_case.py --band 0 --dyn 1
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 3 --csv --log-file gpurun_out/ncu_c4_b32_dyn.csv python tools/prof_case.py --band 32 --dyn 1
timeout 1200 python -m pytest tests/test_gpu_scale.py -x -q 2>&1 | tail -5
