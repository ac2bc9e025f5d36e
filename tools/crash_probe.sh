C=u_512_4_4_128_1024_bf16
for V in '{}' '{"partition_tokens": 2048}' '{"partition_tokens": 512}' '{"smem_stages": 12}' '{"smem_stages": 4}' '{"merge": "combine"}' '{"merge": "cluster"}' '{"kernel": "tc"}'; do
  echo "== $V"
  timeout 120 python tools/one_step.py $C "$V" 2>&1 | tail -2
done
