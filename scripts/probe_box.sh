set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py --steps 2000 --warmup 20 --no-extras > gpurun_out/probe_bench.json 2> gpurun_out/probe_bench.err
tail -c 3000 gpurun_out/probe_bench.json
