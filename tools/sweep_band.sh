# K1 prediction-controller band sweep (PSB_RATIO_BAND=lo,hi), cfg2 shape, eager steps
for band in ${BANDS:-1.08,2.0 1.02,1.5 1.05,1.6 1.1,1.4}; do
  echo "band $band"; PSB_RATIO_BAND=$band PROBE_STEPS=800 python tools/probe_misses.py 2>&1 | tail -1
done
