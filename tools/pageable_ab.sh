show() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['e2e']; print(sys.argv[2], 'pinned %.1f pageable %.1f' % (e['ms_per_step'], e['pageable']['ms_per_step']))" $1 "$2"; }
python bench.py --steps 5 --warmup 3 --no-sparse --no-cpu-baseline > gpurun_out/pg1.json 2>/dev/null; show gpurun_out/pg1.json default
OMP_NUM_THREADS=1 python bench.py --steps 5 --warmup 3 --no-sparse --no-cpu-baseline > gpurun_out/pg2.json 2>/dev/null; show gpurun_out/pg2.json omp1
OPENBLAS_NUM_THREADS=1 python bench.py --steps 5 --warmup 3 --no-sparse --no-cpu-baseline > gpurun_out/pg3.json 2>/dev/null; show gpurun_out/pg3.json blas1
python bench.py --steps 5 --warmup 3 --no-sparse --no-cpu-baseline --no-graph > gpurun_out/pg4.json 2>/dev/null; show gpurun_out/pg4.json nograph
