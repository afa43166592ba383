# compute-sanitizer over tools/sanitize_small.py (every hot kernel at small shapes)
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --kernel-name regex=alise --print-limit 50 \
    python tools/sanitize_small.py > gpurun_out/sanitize_$t.txt 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/sanitize_$t.txt
done
