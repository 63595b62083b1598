set -x
nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null; lscpu | grep -i "model name\|^CPU(s)"
g++ -O2 scratch/hash_threads.cpp paper_2512_17910_b200/build/block_hash.cpp.o -o /tmp/ht -lpthread && /tmp/ht
python scratch/host_time_cpu.py 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_host.json 2> gpurun_out/bench_host.err; tail -c 1500 gpurun_out/bench_host.json
