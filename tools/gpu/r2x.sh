lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core|Flags" | cut -c1-200; grep -o "avx512dq" /proc/cpuinfo | head -1
g++ -O2 -march=x86-64-v3 -std=c++20 -I paper_2603_00326_b200/csrc tools/mb/binom_mb.cpp paper_2603_00326_b200/csrc/host_rng.cpp -o /tmp/binom_mb -pthread
for t in 1 16; do /tmp/binom_mb $t; SOFG_NO_AVX512=1 /tmp/binom_mb $t | tail -1; done
