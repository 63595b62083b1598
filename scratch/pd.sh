

for i in 1 2 3; do echo "epi0: $(timeout 120 python scratch/persist_dbg.py 3000 2048 640 0 2>&1 | tail -1)"; done
for i in 1 2 3; do echo "epi16: $(timeout 120 python scratch/persist_dbg.py 3000 2048 640 16 2>&1 | tail -1)"; done
for i in 1 2 3 4 5; do echo "epi3: $(timeout 120 python scratch/persist_dbg.py 3000 2048 640 3 2>&1 | tail -1)"; done
for i in 1 2 3; do echo "epi2 4096: $(timeout 120 python scratch/persist_dbg.py 3000 4096 640 2 2>&1 | tail -1)"; done
