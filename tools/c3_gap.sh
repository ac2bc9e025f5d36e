# Why is C3 (bf16, GQA 4, P_max 2) slower than C2 (fp16, MHA, P_max 1) at equal bytes?
for r in 1 2; do
python tools/psweep.py c3 '[dict(), dict(partition_tokens=8192), dict(partition_tokens=2048)]'
python tools/psweep.py u_128_32_8_128_8192_fp16 '[dict(), dict(partition_tokens=8192)]'
python tools/psweep.py c2 '[dict(), dict(partition_tokens=2048)]'
python tools/psweep.py u_64_32_32_128_4096_bf16 '[dict()]'
done
