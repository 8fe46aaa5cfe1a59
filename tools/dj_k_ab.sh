for K in 819 1024 2048; do echo "K=$K"; MPSM_DJ_K=$K INTREE=K$K TJOINS=1,16 timeout 300 python tools/merge_variants_run.py; done
