# Hashed N+(v) tables in the clique rows: parity (clique tests) + R-MAT-24 sweep of the knobs.
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -k "clique_bitmap or degeneracy or pair_tail or merge_rows" > gpurun_out/t_nh.log 2>&1; echo rc=$? >> gpurun_out/t_nh.log; tail -2 gpurun_out/t_nh.log
b() { tag=$1; shift; timeout 600 env "$@" > gpurun_out/n_$tag.json 2> gpurun_out/n_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/n_$tag.json 2>&1 | head -3 | cut -c1-330; grep warp-cycles gpurun_out/n_$tag.err | tail -2; }
R24="python bench.py --workload rmat24 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1"
b nh_def $R24
b nh_off GSM_NHASH_MIN=0 $R24
b nh_s32 GSM_CLIQUE_NH_STREAM=32 $R24
b nh_s128 GSM_CLIQUE_NH_STREAM=128 $R24
b nh_s0 GSM_CLIQUE_NH_STREAM=0 $R24
b nh_m8 GSM_NHASH_MIN=8 $R24
b nh_m64 GSM_NHASH_MIN=64 $R24
b nh_T GSM_TRACE=2 $R24
echo nh-done
b nh_hb64k GSM_HUB_BITS=65536 $R24
b nh_hb128k GSM_HUB_BITS=131072 $R24
b nh_hb0 GSM_HUB_BITS=0 $R24
R22="python bench.py --workload rmat22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
b r22_new $R22
b r22_groups GSM_PLAN_GROUPS=1 $R22
echo nh2-done
