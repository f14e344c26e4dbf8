#!/bin/bash
# Development tool: does ptxas keep the constant-bank walk on the uniform datapath (LDCU -> UR operands)
# for a given register cap?  usage: const_ldcu_scan.sh MAXNREG U PART  (PART p = orders 8p+1..8p+8)
cd "$(dirname "$0")/../paper_1904_06229_b200/csrc"
mkdir -p /tmp/ldcu
o=/tmp/ldcu/w_$1_$2_$3.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I. -I../../include \
    -Xptxas -v -DPERM_CONST_ORDERS=0 -DPERM_CONST_MAXNREG_ALL=$1 -DPERM_WALK_U=$2 -DPERM_PART=$3 -c walk_inst.cu -o $o > $o.log 2>&1
for n in $(seq $((8*$3+1)) $((8*$3+8))); do
  if [ $n -gt 48 ] || [ $n -lt 33 ]; then continue; fi
  f="_ZN4perm14walk_kernel_cmILi${n}EEEvNS_11WalkParamsCIXT_EEE"
  c=$(cuobjdump -sass -fun $f $o 2>/dev/null | grep -cE "LDCU.64 UR[0-9]+, c\[0x0\]\[UR")
  s=$(grep -A3 "walk_kernel_cmILi${n}E" $o.log | grep -oE "[0-9]+ bytes spill stores" | head -1)
  echo "n=$n maxnreg=$1 U=$2 ldcu=$c spill=$s"
done
