# K4 level-3 word ranges + keyed-list label index: parity, then A/B bench lines.
python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap or degeneracy or pair_tail or level1 or config or compressed" > gpurun_out/t_perf3.log 2>&1; echo rc=$? >> gpurun_out/t_perf3.log; tail -3 gpurun_out/t_perf3.log
timeout 1500 python -m pytest -x -q tests/test_gpu_configs.py -k "config3 or config4_rmat24_cliques_exact" >> gpurun_out/t_perf3.log 2>&1; echo rc=$? >> gpurun_out/t_perf3.log; tail -3 gpurun_out/t_perf3.log
b() { tag=$1; shift; timeout 900 env "$@" > gpurun_out/q_$tag.json 2> gpurun_out/q_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/q_$tag.json 2>&1 | cut -c1-420; grep -E "warp-cycles|row keys" gpurun_out/q_$tag.err | tail -4; }
b r24 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1
b r24T GSM_TRACE=2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0
b r22 python bench.py --workload rmat22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1
b r22_nolidx GSM_LIDX_MIN=0 python bench.py --workload rmat22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0
b r22_lidx8 GSM_LIDX_MIN=8 python bench.py --workload rmat22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0
b r16 python bench.py --workload rmat16 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0
echo perf3-done
timeout 600 python tools/load_phases.py rmat24 rmat22 > gpurun_out/load_phases.log 2>&1; cat gpurun_out/load_phases.log | tail -40
