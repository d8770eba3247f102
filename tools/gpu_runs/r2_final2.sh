# Round-2 final bench lines (cpu_baseline fixed: spawned oracle passes) + the Fig.-3 sweep.
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
b() { tag=$1; shift; timeout 900 "$@" > gpurun_out/r2_bench_final_$tag.json 2> gpurun_out/r2_bench_final_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/r2_bench_final_$tag.json 2>&1 | head -1 | cut -c1-250; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_final_$tag.json').read().strip().splitlines()[-1]); print('cpu', d.get('cpu_baseline'))"; }
b rmat24 python bench.py
b reference python bench.py --impl reference --steps 3 --warmup 3
b er1000 python bench.py --workload er1000 --steps 20 --warmup 5 --e2e-steps 5
b rmat16 python bench.py --workload rmat16 --steps 5 --warmup 3
b grid1m python bench.py --workload grid1m --steps 5 --warmup 3
b rmat22 python bench.py --workload rmat22 --steps 5 --warmup 3
timeout 2700 python tools/sweep_fig3.py --reps 10 --oracle-s 20 --out gpurun_out/r2_fig3_sweep.jsonl > gpurun_out/r2_fig3.log 2>&1
echo rc=$? >> gpurun_out/r2_fig3.log
tail -3 gpurun_out/r2_fig3.log
echo final2-done
