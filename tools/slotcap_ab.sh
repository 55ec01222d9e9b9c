for sc in 0 1 2; do echo "== DFM_SLOT_CAP=$sc"; DFM_SLOT_CAP=$sc KT_FAMS=1 python tools/kernel_times.py 80 96 112 40; done
for sc in 0 2; do DFM_SLOT_CAP=$sc python tools/opt_ab.py 1 f32 "" | tail -1; done
