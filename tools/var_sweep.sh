# usage: bash tools/var_sweep.sh "<variants>" "<bench rows>" "<python expr over r>"
# A/B of prebuilt libftn variants placed in vtmp/libftn_<name>.so (run under gpurun; "base" = the in-tree build)
cp paper_2409_18824_b200/libftn.so /tmp/libftn_base.so
for v in $1; do
  if [ $v = base ]; then cp /tmp/libftn_base.so paper_2409_18824_b200/libftn.so; else cp vtmp/libftn_$v.so paper_2409_18824_b200/libftn.so; fi
  echo "$v"; python bench.py --rows $2 --no-cpu --steps 6 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['rows']; print($3)"
done
cp /tmp/libftn_base.so paper_2409_18824_b200/libftn.so
