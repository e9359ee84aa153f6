import json,sys
for f in ["gpurun_out/bench_cfg2.log","gpurun_out/bench_cfg5.log"]:
    l=[x for x in open(f) if x.startswith("{")]
    if not l: print(open(f).read()[-2000:]); continue
    j=json.loads(l[-1]); print(f, round(j["ms_per_step"],4), round(j["value"]), {k:round(v["ms"],4) for k,v in j["rooflines"].items()}, "e2e", round(j["e2e"]["ms_per_step"],4))
