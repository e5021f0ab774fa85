# locality relabel in one cooperative kernel: definition test, parity suites using the relabel, config-4/5 builds
set -eo pipefail
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "locality or csr_build or ordered or random_graphs" 2>&1 | tail -1
python -m pytest tests/test_gpu_golden.py -x -q -m gpu -k "c4 or c5" 2>&1 | tail -1
timeout 900 python bench.py --config c4_grid --clusters 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -n 1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('c4', j['config']['phase_ms_rank0'])"
timeout 900 python bench.py --config c5_knn --clusters 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -n 1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('c5', j['config']['phase_ms_rank0'])"
