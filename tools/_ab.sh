for m in 128 256; do
  python tools/level_spmv.py --m $m > gpurun_out/lv_bulk_$m.log 2>&1
  AMGP_LIB=paper_2407_09848_b200/build/variants/libamgp_nobulk.so python tools/level_spmv.py --m $m > gpurun_out/lv_nobulk_$m.log 2>&1
done
