#!/bin/bash
# A/B of two builds of the library (ab_old/, ab_new/) on GEMM shapes, interleaved.
SHAPES=${SHAPES:-"llama_o llama_ffn2 l16_o l16_ffn2 llama_qkv"}
for i in 1 2 3; do
for v in old new; do
python -c "
import sys, runpy; sys.path.insert(0,'.'); sys.argv=['x'] + '$SHAPES'.split()
import paper_2405_05329_b200.kvprefill as kv; kv.LIB_PATH='ab_$v/libkvp_b200.so'
runpy.run_path('scripts/gemm_sweep.py', run_name='__main__')" | python -c "
import sys,json
print('$v', ' '.join(f\"{k}:{v['tflops']:.0f}\" for l in sys.stdin for k,v in json.loads(l).items()))"
done; done
