for env in "LSBA_SPMM_PF=296" "LSBA_SPMM_PF=148" "LSBA_SPMM_PF=592" "LSBA_SPMM_PF=1184" "LSBA_SPMM_PF=296" "LSBA_SPMM_PF=592"; do
  r=$(env $env timeout 400 python bench.py --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs']['spmm'], d['repeats']['GBps'], d['clocks']['sm_mhz'], d['clocks']['power_w'])")
  echo "config 5 [$env]: $r"
done
for env in "LSBA_SPMM_PF=296" "LSBA_SPMM_PF=592" "LSBA_SPMM_PF=1184" "LSBA_SPMM_PF=296"; do
  r=$(env $env timeout 400 python bench.py --config 3 --steps 10 --warmup 3 --repeats 2 --no-cpu-baseline --no-e2e --no-sweep --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['kernel_gbs']['spmm'], d['repeats']['GBps'], d['clocks']['sm_mhz'], d['clocks']['power_w'])")
  echo "config 3 [$env]: $r"
done
