for nt in 256 512 1024; do for rows in 16 32 64 128; do
  v=$(MEGB200_FUSED_NT=$nt MEGB200_FUSED_ROWS=$rows timeout 120 python bench.py --no-cpu-baseline --steps 600 --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['pass_ms']*1e3,1))")
  echo "nt=$nt rows=$rows $v"
done; done
MEGB200_FUSED_NT=1024 MEGB200_FUSED_ROWS=64 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
