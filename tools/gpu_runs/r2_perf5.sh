python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
b() { tag=$1; shift; timeout 900 env "$@" > gpurun_out/v_$tag.json 2> gpurun_out/v_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/v_$tag.json 2>&1 | cut -c1-300; }
R24="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
b def $R24
b noranges GSM_CLIQUE_RANGES=0 $R24
b def2 $R24
b noranges2 GSM_CLIQUE_RANGES=0 $R24
GSM_BIGSORT=0 timeout 600 python tools/load_phases.py rmat24 > gpurun_out/load_nobig.log 2>&1; grep "relabelled\|load 2" gpurun_out/load_nobig.log | tail -3
timeout 600 python tools/load_phases.py rmat24 > gpurun_out/load_big.log 2>&1; grep "relabelled\|load 2" gpurun_out/load_big.log | tail -3
echo perf5-done
