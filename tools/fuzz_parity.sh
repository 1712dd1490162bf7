#!/bin/bash
# usage: tools/fuzz_parity.sh START END [fused]  (restarts after CUDA errors)
k=$1; end=$2; kind=$3
while [ "$k" -lt "$end" ]; do
  out=$(python tools/fuzz_parity.py "$k" "$end" $kind 2>/dev/null)
  echo "$out" | grep -E "^FAIL"
  nxt=$(echo "$out" | grep -E "^RESTART" | awk '{print $2}')
  if [ -z "$nxt" ]; then break; fi
  k=$nxt
done
echo "fuzz done"
