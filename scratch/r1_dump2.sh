rm -f gpurun_out/dump_*.bin
for i in 1 2 3 4 5 6; do SOFG_PROJECT_MODE=0 SOFG_WAVE_DUMP=gpurun_out/dump_$i.bin SOFG_WAVE_HASH=1 python scratch/dbg_hash.py > /dev/null 2>&1; done
md5sum gpurun_out/dump_*.bin
rm -f gpurun_out/dump_*.bin
for i in 1 2 3 4 5 6; do SOFG_PROJECT_MODE=1 SOFG_WAVE_DUMP=gpurun_out/dump_$i.bin SOFG_WAVE_HASH=1 python scratch/dbg_hash.py > /dev/null 2>&1; done
md5sum gpurun_out/dump_*.bin
