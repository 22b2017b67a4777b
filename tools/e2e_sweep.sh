#!/bin/bash
for mb in 4 16 64 256; do
  echo "chunk=${mb}MB"
  IDC_HOST_CHUNK_MB=$mb python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e'])"
done
