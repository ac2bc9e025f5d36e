# e4m3 D split (8 consumer warps, 2 CTAs/SM; PDA_TILE_SPLIT_KV8=1) vs the pair kernel (4 warps, 3 CTAs/SM)
PDA_TILE_SPLIT_KV8=1 python tools/kv8_ts_check.py ts && python tools/kv8_ts_check.py pair && python tools/kv8_ts_check.py cmp
V='[dict(smem_stages=16), dict(smem_stages=24)]'
for r in 1 2; do
for c in c2 c3 c4_b64_ctx4096 c4_b256_ctx4096 u_128_8_1_128_8192_bf16; do
  timeout 300 python tools/psweep.py $c "$V" kv8 | sed 's/^/{"lib": "pair", "r": '$r'} /'
  PDA_TILE_SPLIT_KV8=1 timeout 300 python tools/psweep.py $c "$V" kv8 | sed 's/^/{"lib": "dsplit", "r": '$r'} /'
done
done
PDA_TILE_SPLIT_KV8=1 L2RES_ONCE=0 timeout 120 python tools/l2res.py c2 '[dict(smem_stages=16), dict(smem_stages=24)]' kv8 | sed 's/^/{"lib": "dsplit"} /'
timeout 120 python tools/l2res.py c2 '[dict(smem_stages=16)]' kv8 | sed 's/^/{"lib": "pair"} /'
