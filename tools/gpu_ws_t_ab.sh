for rep in 1 2; do for ws in 0 24 25 33 34; do
  echo "== ws $ws rep $rep"
  python bench.py --config 5 --no-cpu-baseline --no-e2e --secondary "" --steps 20 --warmup 3 --ws $ws 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(r['kernel_ms'], r['frac'])" 2>&1 | tail -1
done; done
python -m pytest tests/test_gpu_bench_paths.py -q -k "full_size and 5" 2>&1 | tail -2
