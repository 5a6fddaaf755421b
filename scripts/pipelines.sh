#!/bin/bash
# The paper's Table 1/2 comparison on the B200 path: every supported
# pipeline x smoother on C0 and C1, each against the reference (oracle/_ref).
#   bash scripts/pipelines.sh OUT.jsonl [configs...]
out=${1:-gpurun_out/pipelines.jsonl}; shift
cfgs=${@:-C0 C1}
for c in $cfgs; do
  for pl in ns_block ns_hybrid2 ns_hybrid1 block; do
    for sm in spai0 ilu0; do
      [ "$pl" = ns_hybrid1 ] && [ "$sm" = ilu0 ] && continue
      python scripts/configs.py $c --ref --pipeline $pl --smoother $sm --out "$out" || echo "FAILED $c $pl $sm"
    done
  done
done
