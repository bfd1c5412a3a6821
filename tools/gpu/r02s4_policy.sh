# GEMM cluster scheduling policy preference (0 default, 1 spread, 2 load balancing)
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
run() { echo "== $1"; for w in 8 5; do env $1 timeout 300 python tools/c3_step.py --world $w --time 2>&1 | tail -1; done
  env $1 timeout 300 python tools/c3_step.py --model 8b --world 1 --time 2>&1 | tail -1; }
for v in FS_GEMM_CLUSTER_POLICY=0 FS_GEMM_CLUSTER_POLICY=1 FS_GEMM_CLUSTER_POLICY=2 FS_GEMM_CLUSTER_POLICY=0; do run "$v"; done
