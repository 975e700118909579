for l in libgsx.so libgsx_ei.so; do
  export GSX_LIB=$PWD/paper_2509_07782_b200/$l
  echo "== $l"
  python -m pytest tests/test_gpu_grad.py -x -q 2>&1 | tail -1
  python profiles/ab_train.py c2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['screen_bwd_logged_ms'], d['plain_bwd_logged_ms'], d['step_ms'])"
  python bench.py --no-cpu-baseline --train-config c4 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', d['train_step']['ms_per_step'], d['train_step']['phases'])"
done
