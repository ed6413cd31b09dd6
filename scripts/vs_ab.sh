# A/B of the one-pass extended frame against the element + merge passes across p (vector_sweep.py):
# mode d = default routing, 1 = LOR_XV=1 (frame wherever it fits), 0 = LOR_XV=0 LOR_XFRAME=0.
mkdir -p gpurun_out
TAG=${VS_TAG:-vs}
for v in d 1 0; do
  if [ $v = d ]; then env -u LOR_XV timeout 900 python scripts/vector_sweep.py ${VS_N:-96} ${VS_SP:-nd,rt,h1} ${VS_P:-1,2,3,4,6} > gpurun_out/${TAG}_x$v.jsonl 2>gpurun_out/${TAG}_x$v.err
  else LOR_XV=$v LOR_XFRAME=$v timeout 900 python scripts/vector_sweep.py ${VS_N:-96} ${VS_SP:-nd,rt,h1} ${VS_P:-1,2,3,4,6} > gpurun_out/${TAG}_x$v.jsonl 2>gpurun_out/${TAG}_x$v.err; fi
  echo "x$v rc=$?"
done
python - <<P
import json
for v in ("d", "1", "0"):
    for l in open(f"gpurun_out/${TAG}_x{v}.jsonl"):
        d=json.loads(l); print(v, d["space"], d["p"], round(d["call_ms"],3), round(d["mdofs"]), d["fill_path"], [round(x,3) for x in d["phases_ms"]])
P
