NGDB_GEMM_FOLD=2 python -m pytest tests/test_gpu_tc_gemm.py -x -q 2>&1 | tail -1
NGDB_GEMM_G2=1 NGDB_GEMM_BN=80 python -m pytest tests/test_gpu_tc_gemm.py -x -q 2>&1 | tail -1
rm -f gpurun_out/gemm_var.jsonl
for v in "80 0 1" "80 1 1" "80 0 2" "80 1 2" "128 0 1" "160 0 1" "160 0 2" "208 0 1" "208 0 2"; do
  set -- $v
  if [ "$2" = "1" ]; then G2=1; else G2=; fi
  NGDB_GEMM_BN=$1 NGDB_GEMM_FOLD=$3 NGDB_GEMM_G2=$G2 python tools/gemm_bench.py | sed "s/\"kernel\": \"[a-z0-9]*\"/\"kernel\": \"bn$1g$2f$3\"/" >> gpurun_out/gemm_var.jsonl
done
python - <<'PY'
import json
rows={}
for l in open("gpurun_out/gemm_var.jsonl"):
  try: d=json.loads(l)
  except: continue
  rows.setdefault(d["shape"],{})[d["kernel"]]=round(d["us"],1)
for k,v in rows.items():
  best=min(v,key=v.get); print(k[:44].ljust(44), best, v)
PY
