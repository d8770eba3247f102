# Spill fix (trace counters to global atomics, 32-bit stats) + filter unroll variants; load phases.
python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap or filter or candidate or long_lists or relabel" > gpurun_out/t_perf4.log 2>&1; echo rc=$? >> gpurun_out/t_perf4.log; tail -3 gpurun_out/t_perf4.log
b() { tag=$1; shift; timeout 900 env "$@" > gpurun_out/u_$tag.json 2> gpurun_out/u_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/u_$tag.json 2>&1 | cut -c1-420; grep -E "warp-cycles|row keys" gpurun_out/u_$tag.err | tail -4; }
b r24 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2
b r24_f1 GSM_FILTER_U=1 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0
b r24_f4 GSM_FILTER_U=4 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0
b r24T GSM_TRACE=2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0
timeout 600 python tools/load_phases.py rmat24 rmat22 > gpurun_out/load_phases.log 2>&1; grep -v "^\[gsm\] k=" gpurun_out/load_phases.log | tail -40
echo perf4-done
