#!/bin/bash
# Development tool: build libperm variants of the n = 44 walk (table path register caps and the
# previous constant-bank walk), for timing with tools/walk_rate.py on the GPU box.
cd "$(dirname "$0")/.."
for R in "$@"; do
  if [ "$R" = "old" ]; then
    PERM_VARIANT=old PERM_EXTRA_FLAGS="-DPERM_TABLE_ORDERS=-1" python -m paper_1904_06229_b200.build &
  else
    PERM_VARIANT=t$R PERM_EXTRA_FLAGS="-DPERM_TABLE_MAXNREG_ALL=$R" python -m paper_1904_06229_b200.build &
  fi
done
wait
