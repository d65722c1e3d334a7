for v in base t128x8 t64x16 t256x8 t128x16; do
  if [ $v = base ]; then L=""; else L="vtmp/libftn_$v.so"; fi
  echo "== $v"; FTN_LIBFTN=$L timeout 300 python tools/prof_tra.py 1024 512 512 20 2>&1
done
for v in t128x8 t256x8; do FTN_LIBFTN=vtmp/libftn_$v.so timeout 600 python -m pytest tests/test_gpu_tra_adv.py -q -x -m "not slow" 2>&1 | tail -1; done
