# round-2 end: GPU suite, smoke, default bench, reference arm, then the records refresh
bash scripts/r2_final.sh
bash scripts/r2_records_final.sh
