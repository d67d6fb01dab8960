#!/bin/bash
# ncu --set full of the final attention kernels: persistent chunk-frame (after the O offload) and the decode
# kernel over a chunk-frame wave (per-frame q rotation)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3f
N="ncu --profile-from-start off --clock-control none"
timeout 900 $N --set full --import-source on -k regex:attn_qp -c 1 -o gpurun_out/s3f/ncu_attn_qp python scripts/ncu_link.py --config cfg4 --layers 2 > gpurun_out/s3f/a.log 2>&1
DECODE_FRAMES=1 DECODE_NCU=1 timeout 900 $N --set full --import-source on -k regex:attn_decode -c 1 -o gpurun_out/s3f/ncu_attn_decode_frames python scripts/decode_profile.py 32 1 > gpurun_out/s3f/d.log 2>&1
for f in ncu_attn_qp ncu_attn_decode_frames; do python scripts/ncu_detail.py gpurun_out/s3f/$f.ncu-rep > gpurun_out/s3f/$f.md 2>&1; head -22 gpurun_out/s3f/$f.md; done
