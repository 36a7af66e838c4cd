#!/bin/bash
# What ONE GPU can measure of the P-rank strong-scaling run of config 5 (this
# pool has one GPU per call): the per-rank step at the P-rank size.  `bench.py --rank-proxy P`
# runs the stencil on one rank's slab (256 x 256 x 256/P, the same rows, nonzeros per row and
# block sizes as that rank's share; the neighbours' planes are cut off instead of exchanged) as
# a one-rank problem, here through the distributed code path with a real one-rank NCCL
# communicator (LSBA_FORCE_COMM=1: halo/allreduce launches, identical-enqueue rule), with the
# Gram allreduce as ncclAllReduce (LSBA_DEVAR=0) or inside the Gram tail (f2, LSBA_DEVAR=1).
# Not measured here: the halo's wire time (overlapped with the interior rows by design) and the
# cross-GPU latency of the allreduce.  E_kernel(P) = steps/s(slab) / (P * steps/s(P = 1)) is
# therefore an UPPER bound of the strong-scaling efficiency: what the kernels alone allow.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/rank_proxy.txt
: > $out
line() {  # $1 = label, rest = env + bench args
  local label="$1"; shift
  r=$(env "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%s | n=%d | %.1f block steps/s | %.1f us/step | %.0f GB/s | %.1f%% of HBM | launches %d | SM %s MHz %s' % (d['config']['workload'], d['config']['n'], d['block_steps_per_s'], 1e3*d['ms_per_block_step'], d['value'], 100*d['pct_roofline']['of_measured_hbm'], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons']))" 2>&1)
  echo "[$label] $r" | tee -a $out
}
COMMON="--config 5 --steps 3 --warmup 2 --repeats 3 --no-cpu-baseline --no-e2e --no-sweep --no-tts"
line "P=1 one-rank path" LSBA_FORCE_COMM=0 timeout 600 python bench.py $COMMON
for P in ${PROXY_P:-2 4 8}; do
  line "P=$P slab, one-rank path"        LSBA_FORCE_COMM=0 timeout 600 python bench.py $COMMON --rank-proxy $P
  line "P=$P slab, NCCL path, DEVAR=0"   LSBA_FORCE_COMM=1 LSBA_DEVAR=0 timeout 600 python bench.py $COMMON --rank-proxy $P
  line "P=$P slab, NCCL path, DEVAR=1"   LSBA_FORCE_COMM=1 LSBA_DEVAR=1 timeout 600 python bench.py $COMMON --rank-proxy $P
done
