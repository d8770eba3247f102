python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap or degeneracy" > gpurun_out/t_perf6.log 2>&1; echo rc=$? >> gpurun_out/t_perf6.log; tail -3 gpurun_out/t_perf6.log
timeout 1200 python -m pytest -x -q tests/test_gpu_configs.py -k "config4_rmat24_cliques_exact" >> gpurun_out/t_perf6.log 2>&1; echo rc=$? >> gpurun_out/t_perf6.log; tail -3 gpurun_out/t_perf6.log
b() { tag=$1; shift; timeout 900 env "$@" > gpurun_out/w_$tag.json 2> gpurun_out/w_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/w_$tag.json 2>&1 | cut -c1-300; }
R24="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
b def $R24
b hb128k GSM_HUB_BITS=131072 $R24
b hb32k GSM_HUB_BITS=32768 $R24
b noranges GSM_CLIQUE_RANGES=0 $R24
echo perf6-done
