for i in 1 2 3 4 5 6; do
  echo "== run $i"
  CHAM_LIB=$PWD/build/lib_dbg.so timeout 100 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dbg_$i.txt 2>&1
  grep -E "DBG" gpurun_out/dbg_$i.txt | sort | uniq -c | sort -rn | head -8
  tail -1 gpurun_out/dbg_$i.txt | cut -c1-120
done
