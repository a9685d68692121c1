import io, sys, json, gzip
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2404_19391_b200 as z
from test_gpu_parity import dict_from_json
cases=json.load(gzip.open('tests/golden/stream_cases.json.gz'))
dicts=[dict_from_json(dj) for dj in cases["dicts"]]
nbad=0
for i,c in enumerate(cases["cases"]):
    if "err" in c: continue
    dst=io.BytesIO()
    st=z.run_stream(io.BytesIO(bytes.fromhex(c["payload"])), dst, dicts[c["dict"]], c["direction"], preprocess=c["preprocess"], lenient=c["lenient"])
    got=dst.getvalue(); want=bytes.fromhex(c["out"])
    if got!=want:
        nbad+=1
        if nbad<=3:
            pay=bytes.fromhex(c["payload"])
            gl=got.split(b'\n'); wl=want.split(b'\n'); pl=pay.split(b'\n')
            print("case",i,c["direction"],"pre",c["preprocess"],"len",c["lenient"],"dict",c["dict"], "nlines",len(pl), len(gl), len(wl))
            for k,(a,b) in enumerate(zip(gl,wl)):
                if a!=b:
                    print(" line",k,"in",pl[k] if k<len(pl) else None); print("  got ",a); print("  want",b); break
print("bad",nbad)
