#!/bin/bash
# e2e (host buffers) of the default workload for several host chunk sizes
for mb in ${SWEEP_MB:-16 32 64 128}; do
  echo "chunk=${mb}MB"
  IDC_HOST_CHUNK_MB=$mb python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])"
done
