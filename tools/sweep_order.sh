#!/bin/bash
# side-stream launch order of the four type kernels (HW_TYPE_ORDER, run time) at N=4/5
for n in 4 5; do
  for o in 2013 3012 0123 3210 2310 0213; do
    echo -n "N=$n order=$o "; HW_TYPE_ORDER=$o tools/quick.sh --order $n
  done
done
