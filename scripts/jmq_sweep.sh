for q in 8 16 33 37 64; do
  echo "Q=$q"
  CDN_JDEBUG=1 CDN_JMQ=$q JM_ONLY=1 JM_LAYERS=C5:0,C5:2 timeout 200 python scripts/jm_probe.py 8 32 2>&1 | grep -v "^\[cdn\] joint layer"
done
