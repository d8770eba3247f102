# Round-2 measurement pass: order variants of the clique path, the north_star's breadth-first
# path on configs[4], ENUMERATE lines, look-ahead / compressed ablations, shard balance.
# Every bench line -> gpurun_out/m_<tag>.json (stderr .err); summary -> stdout.
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py -k "degeneracy" > gpurun_out/t_order.log 2>&1; echo rc=$? >> gpurun_out/t_order.log
tail -2 gpurun_out/t_order.log
b() { tag=$1; shift; timeout 900 env "$@" > gpurun_out/m_$tag.json 2> gpurun_out/m_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/m_$tag.json 2>&1 | tail -4; grep "warp-cycles" gpurun_out/m_$tag.err | tail -2; }
b deg python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1
b adg GSM_ORDER=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1
b degT GSM_TRACE=2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0
b adgT GSM_TRACE=2 GSM_ORDER=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0
b bfs24 python bench.py --steps 3 --warmup 3 --clique 0 --no-cpu-baseline --e2e-steps 0
b bfs24c python bench.py --steps 3 --warmup 3 --clique 0 --compressed --no-cpu-baseline --e2e-steps 0
b rmat22 python bench.py --workload rmat22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1
b er1000 python bench.py --workload er1000 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1
b enum16 python bench.py --workload rmat16 --mode enumerate --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1
b enumgrid python bench.py --workload grid1m --mode enumerate --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1
b grid_la0 python bench.py --workload grid1m --steps 5 --warmup 3 --lookahead 0 --clique 0 --no-cpu-baseline --e2e-steps 0
b grid_la1 python bench.py --workload grid1m --steps 5 --warmup 3 --lookahead 1 --clique 0 --no-cpu-baseline --e2e-steps 0
b grid_la2 python bench.py --workload grid1m --steps 5 --warmup 3 --lookahead 2 --clique 0 --no-cpu-baseline --e2e-steps 0
timeout 900 python tools/shard_balance.py --workload rmat24 --shards 8 > gpurun_out/shard_rmat24.json 2> gpurun_out/shard_rmat24.err
timeout 900 python tools/shard_balance.py --workload rmat22 --shards 8 > gpurun_out/shard_rmat22.json 2> gpurun_out/shard_rmat22.err
tail -c 600 gpurun_out/shard_rmat24.json; tail -c 600 gpurun_out/shard_rmat22.json
echo measure-done
