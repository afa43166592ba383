set -x
for ppc in 0 32 64; do timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-pred --no-c5 --no-c3 --planes-per-chunk $ppc > gpurun_out/bench71_$ppc.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench71_$ppc.json')); print($ppc, d['value'], d['roofline_link']['frac'], d['roofline_link']['peak'])"; done
