# Knob sweeps: pair-tail membership variants on configs[3] (round-1 129 ms vs 284 ms now),
# hub bitmap size / ratio on configs[4].
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
b() { tag=$1; shift; timeout 600 env "$@" > gpurun_out/p_$tag.json 2> gpurun_out/p_$tag.err; echo "== $tag $*"; python tools/show_bench.py gpurun_out/p_$tag.json 2>&1 | head -1 | cut -c1-400; }
R22="python bench.py --workload rmat22 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0"
R24="python bench.py --workload rmat24 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0"
b r22_def $R22
b r22_nohub GSM_MEMBER_HUB=0 $R22
b r22_noswap GSM_MEMBER_SWAP=0 $R22
b r22_nohub_noswap GSM_MEMBER_HUB=0 GSM_MEMBER_SWAP=0 $R22
b r22_nogroups GSM_PLAN_GROUPS=0 $R22
b r22_none GSM_MEMBER_HUB=0 GSM_MEMBER_SWAP=0 GSM_PLAN_GROUPS=0 $R22
b r22_hb0 GSM_HUB_BITS=0 $R22
b r22_pt8 GSM_PAIR_THREAD_MAX=8 $R22
b r22_pt32 GSM_PAIR_THREAD_MAX=32 $R22
b r24_hb0 GSM_HUB_BITS=0 $R24
b r24_hb16k GSM_HUB_BITS=16384 $R24
b r24_hb48k GSM_HUB_BITS=49152 $R24
b r24_hb64k GSM_HUB_BITS=65536 $R24
b r24_r16 GSM_CLIQUE_HUB_RATIO=16 $R24
b r24_r256 GSM_CLIQUE_HUB_RATIO=256 $R24
b r24_s64 GSM_CLIQUE_STREAM=64 $R24
b r24_s256 GSM_CLIQUE_STREAM=256 $R24
echo perf2-done
