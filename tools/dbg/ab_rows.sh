# Row windows vs flat vectors on the short-odd-row shape zoo, same box (tools/dbg/ab_table.py
# prints the comparison).  profiles/r01_rows_sweep.jsonl holds the windows-per-group /
# minimum-chunk sweep measured while tuning the plan's defaults.
python tools/shape_zoo.py --rows | sed 's/^{/{"lib": "rows", /'
python tools/shape_zoo.py --rows --policy 5,0 | sed 's/^{/{"lib": "flat", /'
