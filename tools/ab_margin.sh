# A/B of the warm-start margins and evict-first eps stores (EF steady state)
for rep in 1 2 3; do
  for v in main lo128 hi16 epsef; do
    if [ $v = main ]; then L=paper_1802_08021_b200/libsparcml.so; else L=paper_1802_08021_b200/libvar_$v.so; fi
    echo "== topk $v" >> gpurun_out/mg_ab.log
    SPARCML_LIB=$L timeout 60 python tools/topk_phases.py --pre 80 --reps 40 >> gpurun_out/mg_ab.log 2>&1
  done
done
