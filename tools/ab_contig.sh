# access granularity: shuffled vs contiguous block placement, 16-bit vs e4m3 slabs
for c in c2 c3; do
python tools/psweep.py $c '[dict()]'
PSWEEP_CONTIGUOUS=1 python tools/psweep.py $c '[dict()]'
python tools/psweep.py $c '[dict()]' kv8
PSWEEP_CONTIGUOUS=1 python tools/psweep.py $c '[dict()]' kv8
done
