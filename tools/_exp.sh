for cfg in "4 32" "2 64" "2 96" "4 48" "1 128" "8 32"; do
  set -- $cfg
  echo CH=$1 NSTW=$2 $(EGT_WIDE_CH=$1 EGT_WIDE_NSTW=$2 python tools/verify_probe.py 80 8 2>&1 | grep M=) $(EGT_WIDE_CH=$1 EGT_WIDE_NSTW=$2 python tools/verify_probe.py 272 8 2>&1 | grep M=)
done
