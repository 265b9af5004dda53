import json, sys
for v in sys.argv[1:]:
    try:
        d = json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
        print(v, round(d["ms_per_step"], 3), {k: round(x, 3) for k, x in d["phases_ms"].items()})
    except Exception as e:
        print(v, "ERR", open(f"gpurun_out/var_{v}.json").read()[-500:])
