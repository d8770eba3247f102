# Round-2: parity of the latest kernels, then one `ncu --set full` capture per hot kernel,
# each reduced ON THE BOX to a text brief (details + top source lines) and a raw-page CSV;
# the .ncu-rep files are deleted (gpurun copies back at most 64 MiB of gpurun_out/).
python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap or degeneracy or merge_rows or level1 or pair_tail" > gpurun_out/t_full2.log 2>&1; echo rc=$? >> gpurun_out/t_full2.log; tail -3 gpurun_out/t_full2.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; python tools/show_bench.py gpurun_out/f2_bench.json | cut -c1-400
B() { echo "python bench.py --workload $1 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 $2"; }
# F tag kernel-regex launch-skip workload [bench args]
F() {
  tag=$1; rx=$2; sk=$3; wl=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" --launch-skip $sk -c 1 \
      -o gpurun_out/full_$tag $(B $wl "$*") > gpurun_out/ncu_full_$tag.log 2>&1
  echo "full $tag rc=$?"
  if [ -f gpurun_out/full_$tag.ncu-rep ]; then
    python tools/ncu_brief.py gpurun_out/full_$tag.ncu-rep 30 > gpurun_out/r2_ncu_full_${tag}_brief.txt 2>&1
    ncu -i gpurun_out/full_$tag.ncu-rep --page raw --csv > gpurun_out/r2_ncu_full_${tag}_raw.csv 2>/dev/null
    rm -f gpurun_out/full_$tag.ncu-rep
  fi
}
F k3_cta256 "k_clique_cta" 3 rmat24
F k4_cta1024 "k_clique_cta" 7 rmat24
F k3_warp "k_clique_warp" 0 rmat24
F filter24 "k_filter" 0 rmat24
F pair22 "k_pair<" 0 rmat22
F plan22 "k_plan_rows" 0 rmat22
F refine22 "k_refine" 0 rmat22 --refine-rounds 1
F expand16 "k_expand" 0 rmat16
F walk16 "k_count_walk" 0 rmat16
F tail24 "k_tail" 0 rmat24 --clique 0
du -sh gpurun_out
echo full2-done
