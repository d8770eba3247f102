# Round-2 checkpoint on the GPU: full GPU suite + smoke, default bench line, configs[3] compressed
# + level-1 shard balance, configs[0..2] lines.
python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log; tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
b() { tag=$1; shift; timeout 900 env "$@" > gpurun_out/c_$tag.json 2> gpurun_out/c_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/c_$tag.json 2>&1 | cut -c1-420; }
b default python bench.py
b rmat22 python bench.py --workload rmat22 --steps 5 --warmup 3 --e2e-steps 2
b rmat22c python bench.py --workload rmat22 --steps 5 --warmup 3 --compressed --no-cpu-baseline --e2e-steps 0
b er1000 python bench.py --workload er1000 --steps 20 --warmup 5 --e2e-steps 3
b rmat16 python bench.py --workload rmat16 --steps 5 --warmup 3 --e2e-steps 2
b grid1m python bench.py --workload grid1m --steps 5 --warmup 3 --e2e-steps 2
timeout 900 python tools/shard_balance.py --workload rmat22 --shards 8 --level1 > gpurun_out/shard_rmat22_l1.json 2> gpurun_out/shard_rmat22_l1.err; tail -c 400 gpurun_out/shard_rmat22_l1.json
echo round-done
