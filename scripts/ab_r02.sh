L=paper_2411_10958_b200
python scripts/kernel_ab.py 32768 128 v8,v13,v13@$L/libsage2_ks3.so,v13@$L/libsage2_pc16.so 3
python scripts/kernel_ab.py 32768 64 v12,v13,v13@$L/libsage2_ks3.so,v13@$L/libsage2_pc16.so 3
python scripts/kernel_ab.py 4096 64 v12,v8,v13 3
python scripts/kernel_ab.py 4096 64 v8_causal,v13_causal 3
python scripts/kernel_ab.py 1024 64 v12,v8,v13 5
python scripts/kernel_ab.py 1024 128 default,v8,v13 5
python scripts/kernel_ab.py 1024 128 v8_causal,v13_causal 5
python scripts/kernel_ab.py 16384 64 v8_causal,v13_causal 3
