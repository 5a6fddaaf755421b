#!/bin/bash
# The paper's Table 1/2 comparison (Scalar, Block,
# NS Scalar, NS Hybrid1, NS Hybrid2, NS Block with ILU(0)) on the B200 path,
# each against the reference (oracle/_ref) on the same problem: setup /
# solve seconds, iterations, preconditioner bytes, hierarchy bit-identity.
#   bash scripts/pipelines.sh OUT.jsonl [configs...]
out=${1:-gpurun_out/pipelines.jsonl}; shift
cfgs=${@:-C0 C1}
for c in $cfgs; do
  for pl in scalar block ns_scalar ns_hybrid1 ns_hybrid2 ns_block; do
    python scripts/configs.py $c --ref --pipeline $pl --smoother ilu0 --out "$out" || echo "FAILED $c $pl ilu0"
  done
done
