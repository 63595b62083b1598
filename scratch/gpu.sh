#!/bin/bash
# Build in-tree; only on success ship the snapshot to a B200 and run "$1" there.
set -e
cd /root/repo
make -C /root/repo/paper_2512_17910_b200 -j8 > /tmp/build.log 2>&1 || { grep -E "error" -A3 /tmp/build.log | head -30; exit 1; }
grep -h -A2 "${KERNEL_RE:-attn_tc_kernel}" paper_2512_17910_b200/build/*.ptxas.log 2>/dev/null | grep -E "registers|spill" | head -4 || true
timeout "${OUTER:-1800}" /usr/local/graft/bin/gpurun --timeout "${LIMIT:-600}" -- "$1" 2>&1 | grep -v "^\[gpurun\] sending"
