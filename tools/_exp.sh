export EGT_BENCH_NO_VERIFY=1
python tools/decode_probe.py int4-2:4
EGT_DECODE_NO_L2PF=1 python tools/decode_probe.py int4-2:4
