# ncu capture + in-kernel timeline of the config-4 FlashAssign (ALT path).
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:fk_assign_tc2 -s 3 -c 1 -o gpurun_out/cfg4_assign -f \
  python scripts/assign_time.py 64 16384 256 64 float16 1 > gpurun_out/cfg4_assign.log 2>&1
FK_ASSIGN_TRACE=gpurun_out/trace_cfg4.txt python scripts/assign_time.py 64 16384 256 64 float16 1 >> gpurun_out/cfg4_assign.log 2>&1
