timeout 300 python tools/gpu/k5ab.py paper_1203_5128_b200/libsbf_head.so paper_1203_5128_b200/libsbf.so
timeout 300 python tools/gpu/dbg_split2.py 2>&1 | grep -v Warn | grep -v "res = P" | tail -12
