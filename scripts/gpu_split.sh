export CUDA_MODULE_LOADING=EAGER
for sp in 37 9 18 74 148; do
  echo "splits $sp"; FC_SPLITS=$sp timeout -s KILL 200 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -2
  FC_SPLITS=$sp timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_shortlist_pair -s 2 -c 1 python scripts/time_lookup.py 1000000 32 768 2>&1 | grep -E "dram__bytes_read.sum|gpu__time_duration|lts__t_sector_hit" 
done
