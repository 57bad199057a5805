import json
for l in open("gpurun_out/ab.txt"):
    n,j=l.split(" ",1); d=json.loads(j)["k_trace_query"]; print(n, {k:round(v["ms"],3) for k,v in d.items()})
