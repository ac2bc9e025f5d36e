# one-wave split cells: 8 vs 12 ring stages, and the 4-CTA cluster case (u_74 ctx 16k) -- occupancy / DRAM
bash tools/ncu_quick.sh g_u128_s8 splitk_kernel python tools/one_step.py u_128_8_1_128_8192_bf16
bash tools/ncu_quick.sh g_u128_s12 splitk_kernel python tools/one_step.py u_128_8_1_128_8192_bf16 '{"smem_stages": 12}'
bash tools/ncu_quick.sh g_u148_s8 splitk_kernel python tools/one_step.py u_148_8_1_128_8192_bf16
bash tools/ncu_quick.sh g_u74 splitk_kernel python tools/one_step.py u_74_8_1_128_16384_bf16
bash tools/ncu_quick.sh g_c2 splitk_kernel python tools/one_step.py c2
