# Attention variant sweep: correctness (gpu parity tests) per variant, then TTFT/attention TF/s.
# usage: bash scripts/attn_sweep.sh "wpq:poly ..." "workloads..."
VARIANTS=${1:-"1:0 2:0 1:4 1:6"}
WORKLOADS=${2:-"llama7b-4k llama7b-16k falcon7b-8k"}
mkdir -p gpurun_out
for v in $VARIANTS; do
  export KVP_ATTN_WPQ=${v%%:*} KVP_ATTN_POLY=${v##*:}
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "attention or golden or bf16" 2>&1 | tail -2 | sed "s/^/[$v] /"
  for w in $WORKLOADS; do
    timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['attention']; print('[$v] $w ttft %.2f ms attn %.3f ms %.0f TF/s clk %s' % (d['value'], k['ms'], k['tflops'], d['clocks']['sm_mhz']))"
  done
done
