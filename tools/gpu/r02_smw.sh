python tools/dec_smweight.py; DEC_SHAPE=5,80,8,8,64,4096 python tools/dec_smweight.py; DEC_SHAPE=1,32,8,4,64,4096 python tools/dec_smweight.py
