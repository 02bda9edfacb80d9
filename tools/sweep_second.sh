# second-chance factor x controller band (tools/probe_misses.py, 800 eager cfg2 steps each)
for f2 in ${F2S:-0 0.9 0.95 0.97}; do
  for band in ${BANDS:-1.08,2.0 1.05,1.6 1.02,1.5}; do
    echo "f2 $f2 band $band: $(PSB_SECOND_F=$f2 PSB_RATIO_BAND=$band PROBE_STEPS=800 python tools/probe_misses.py 2>&1 | tail -1)"
  done
done
