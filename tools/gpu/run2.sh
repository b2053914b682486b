set -x
export PYTHONUNBUFFERED=1
for i in 1 2; do
CHEBFD_B200_LIB=$PWD/build/ab/libchebfd_r01.so timeout 600 python tools/band_exp.py --cases c2,c4 --bytes -1 --deg 60
timeout 600 python tools/band_exp.py --cases c2,c4 --bytes 0,16 --deg 60
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 python tools/prof_case.py --band 0 && \
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 4 --csv --log-file gpurun_out/ncu_c4_band0.csv python tools/prof_case.py --band 0
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 4 --csv --log-file gpurun_out/ncu_c4_band16.csv python tools/prof_case.py --band 16
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 4 --csv --log-file gpurun_out/ncu_c4_band64.csv python tools/prof_case.py --band 64
ncu --metrics $M --clock-control none -k regex:step_tma -s 2 -c 4 --csv --log-file gpurun_out/ncu_c2.csv python tools/prof_case.py --lattice 64 64 64 --nb 32
