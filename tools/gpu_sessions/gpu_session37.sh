for f in 0 0.5 1.0; do QAA_PERSIST_L2=$f timeout 120 python tools/diag_super2.py 1 20 30; done
for f in 0 1.0; do QAA_PERSIST_L2=$f timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qaa_superpass -s 4 -c 2 python tools/diag_super2.py 1 4 30 2>&1 | grep -E "dram__|duration|persisting"; done
