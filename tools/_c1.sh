for b in 4 6 8; do echo "bands $b: $(HSDLA_B200_BANDS=$b python tools/small_probe.py c2 --calls 12 | cut -c1-44 | tr '\n' ' ')"; done
for b in 2 3 4; do echo "bands $b: $(HSDLA_B200_BANDS=$b python tools/small_probe.py s3 --calls 12 | cut -c1-44 | tr '\n' ' ')"; done
