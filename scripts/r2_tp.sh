cd $GRAFT_REPO_ROOT
for lib in libpic.so libpic_2p.so; do
PIC_LIB_NAME=$lib PIC_ATTN_TRACE=1 timeout 600 python scripts/ncu_link.py --config cfg4 --layers 2 --graph 0 --kv-share 0 2>&1 | grep "attn_pp" | tail -21 | grep "span\|compute\|wait S" ; echo "== $lib"
done
