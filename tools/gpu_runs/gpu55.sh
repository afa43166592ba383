set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench55.json 2> gpurun_out/bench55.err; tail -2 gpurun_out/bench55.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench55_ref.json 2>&1; tail -1 gpurun_out/bench55_ref.json | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
