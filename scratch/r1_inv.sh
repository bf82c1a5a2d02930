for i in 1 2 3 4; do SOFG_PROJECT_MODE=1 SOFG_DEBUG_INV=1 SOFG_WAVE_HASH=1 python scratch/dbg_hash.py > gpurun_out/inv_$i.log 2>&1; done
for i in 2 3 4; do diff gpurun_out/inv_1.log gpurun_out/inv_$i.log | head -6; echo ---; done
