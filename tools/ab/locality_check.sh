set -o pipefail
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "locality_order" 2>&1 | tail -1
timeout 900 python tools/locality_check.py c5_knn
timeout 900 python tools/locality_check.py c4_grid
timeout 900 python bench.py --config c5_knn --clusters 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -n 1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('c5', j['config']['phase_ms_rank0'])"
