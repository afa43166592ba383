# launch list of the bench command, our kernels only (ncu -k filter), for kernel shares
set -x
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 3000 --csv --log-file gpurun_out/launches28.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-c5 > gpurun_out/ncu28.log 2>&1; echo ncu $?
tail -3 gpurun_out/ncu28.log
