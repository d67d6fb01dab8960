#!/bin/bash
cd $GRAFT_REPO_ROOT
for lib in libpic_k2.so libpic.so libpic_k2.so libpic.so; do
PIC_LIB_NAME=$lib PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share 0 2>&1 | grep -E "CTA span|smA compute" | tail -2; echo "== $lib"
done
