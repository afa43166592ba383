ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 1000000 256 2>&1 | grep "rescore q=" | awk '{for(i=1;i<=NF;i++) if($i=="dots") d=$(i+1); if (d>40000) print}' | head -8
ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 1000000 256 2>&1 | grep -c "rescore q="
