# A/B: programmatic dependent launch (PDA_PDL=1) vs plain launches, back-to-back steps
for r in 1 2; do
  echo "PDL1 $(PDA_PDL=1 python tools/floor.py c1 c4_b1_ctx512 c4_b16_ctx512 c4_b4_ctx4096 c4_b64_ctx512 c4_b64_ctx4096 2>/dev/null | tr '\n' ' ')"
  echo "PDL0 $(PDA_PDL=0 python tools/floor.py c1 c4_b1_ctx512 c4_b16_ctx512 c4_b4_ctx4096 c4_b64_ctx512 c4_b64_ctx4096 2>/dev/null | tr '\n' ' ')"
done
for r in 1 2; do
  echo "BENCH PDL1 $(PDA_PDL=1 python bench.py --no-extras --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["us_per_step"])')"
  echo "BENCH PDL0 $(PDA_PDL=0 python bench.py --no-extras --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["us_per_step"])')"
  echo "BENCH C3 PDL1 $(PDA_PDL=1 python bench.py --config c3 --no-extras --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["us_per_step"])')"
  echo "BENCH C3 PDL0 $(PDA_PDL=0 python bench.py --config c3 --no-extras --steps 50 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["us_per_step"])')"
done
