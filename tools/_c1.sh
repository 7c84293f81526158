python tools/quick_bench.py c1 c2 c3 2>&1 | grep merged | cut -c1-75
python tools/sweep.py --only c5_na16_ng2000,c5_na64_ng2000,c5_na256_ng2000,c5_na64_ng5000,c5_na64_ng10000,c2 --out gpurun_out/sw.jsonl 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['point'], round(d['build_ms'], 3), round(d['tflops'], 2), round(d['executed_frac_of_dmma_peak'], 3))"
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not unmodified_reference and not config3" 2>&1 | tail -2
