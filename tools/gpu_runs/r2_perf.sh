# Round-2 quick perf: clique path variants on R-MAT-24 (hub bitmap size / ratio), one bench line each.
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/perf_$tag.json 2> gpurun_out/perf_$tag.err; python - "$tag" <<'PY'
import json,sys
tag=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/perf_{tag}.json").read().strip().splitlines()[-1])
    pq=d["per_query_rank0"]
    print(tag, "ms/step %.1f" % d["ms_per_step"], {k: round(v["ms"]["total"],1) for k,v in pq.items()}, {k: v["unique"] for k,v in pq.items()})
except Exception as e:
    print(tag, "FAILED", e, open(f"gpurun_out/perf_{tag}.err").read()[-800:])
PY
}
run nohub GSM_HUB_BITS=0
run hub32k GSM_HUB_BITS=32768
run hub16k GSM_HUB_BITS=16384
run hub64k GSM_HUB_BITS=65536
run hub32k_r32 GSM_HUB_BITS=32768 GSM_CLIQUE_HUB_RATIO=32
run hub32k_r256 GSM_HUB_BITS=32768 GSM_CLIQUE_HUB_RATIO=256
run hub32k_r16 GSM_HUB_BITS=32768 GSM_CLIQUE_HUB_RATIO=16
echo perf-done
