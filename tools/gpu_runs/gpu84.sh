set -x
for B in 256 64 1; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches84_b$B.csv python tools/pred_bench.py 1000000 $B > /dev/null 2>&1; echo ncu $?
python tools/launch_share.py gpurun_out/launches84_b$B.csv | head -14
done
