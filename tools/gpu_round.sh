# Round validation on a B200 box: GPU tests, bench (own + reference arm), smoke.
# usage: gpurun -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-run}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.txt
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
cat gpurun_out/${TAG}_pytest.txt; tail -3 gpurun_out/${TAG}_bench.err; tail -1 gpurun_out/${TAG}_smoke.txt
