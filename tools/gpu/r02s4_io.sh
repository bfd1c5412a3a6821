for v in graph api graph api; do FS_E2E_IO=$v python bench.py --skip-failure-states --skip-recovery --skip-cpu --skip-mixed --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
