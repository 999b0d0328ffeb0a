echo new; python tools/blk_dec_ab.py
echo old; A8_BLK_DEC_TMA=0 python tools/blk_dec_ab.py
