#!/bin/bash
# usage: tools/fuzz_parity.sh START END [fused]  (restarts after CUDA errors)
# prints every FAIL line, then "checked A..B" for each process that reached
# its end (a run that never prints it did not finish)
k=$1; end=$2; kind=$3
while [ "$k" -lt "$end" ]; do
  out=$(python tools/fuzz_parity.py "$k" "$end" $kind 2>&1)
  echo "$out" | grep -E "^FAIL"
  echo "$out" | grep -E "^DONE" | sed "s/^DONE/checked $k../"
  nxt=$(echo "$out" | grep -E "^RESTART" | awk '{print $2}')
  if [ -z "$nxt" ]; then
    echo "$out" | grep -qE "^DONE|^RESTART" || { echo "fuzz process failed:"; echo "$out" | tail -5; }
    break
  fi
  k=$nxt
done
echo "fuzz done"
