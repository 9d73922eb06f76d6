for G in 2 4 8; do
  python scripts/probe_g8.py --G $G --S 1024 2>&1 | grep -E "^G=|seg|bag_fwd|total"
  ML_SEG_PIPE=0 python scripts/probe_g8.py --G $G --S 1024 2>&1 | grep -E "seg_|total"
done
