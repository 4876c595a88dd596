for v in default s3 pp4; do
  for r in 1 2; do
    HIPATTN_MASK_TC=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['mask_ms'], d['attn_ms'])"
  done
done
HIPATTN_MASK_TC=s3 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 s3', d['mask_ms'], d['attn_ms'])"
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 default', d['mask_ms'], d['attn_ms'])"
