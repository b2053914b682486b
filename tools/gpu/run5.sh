set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -3
CHEBFD_B200_LIB=$PWD/build/ab/libchebfd_r01.so timeout 600 python tools/band_exp.py --cases c2,c4,c3_256,c3_32 --bytes -1 --deg 60
timeout 1200 python tools/band_exp.py --cases c2,c4,c3_256,c3_32 --bytes 0,8,16,32 --dyn 1,2,4 --deg 60
CHEBFD_B200_LIB=$PWD/build/ab/libchebfd_r01.so timeout 600 python tools/band_exp.py --cases c2,c4 --bytes -1 --deg 60
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 600 python tools/prof_case.py --band 16 --dyn 2 && \
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 3 --csv --log-file gpurun_out/ncu_c4_b16_tpc2.csv python tools/prof_case.py --band 16 --dyn 2
