# L2 bulk prefetch of each iteration's representative rows: off vs on (decode, C2, C4, C5)
for pf in 0 1; do
  HIPATTN_PREFETCH=$pf timeout 120 python bench.py --decode-only 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf=$pf decode', d['mask_us'], d['attn_us'], d['options']['gqa_shared_chunks4']['mask_us'])"
  for c in c2 c4; do
    HIPATTN_PREFETCH=$pf timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf=$pf $c', d['mask_ms'], d['attn_ms'])"
  done
  HIPATTN_PREFETCH=$pf timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-extras --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pf=$pf c5', d['mask_ms'], d['attn_ms'])"
done
