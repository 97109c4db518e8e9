# decode GEMM configuration sweep (GPU box)
python tools/dec_gemm_sweep.py
for sp in 1 2 4 8; do NMT_DEC_SPLITS=$sp python tools/dec_gemm_sweep.py; done
for t in 128 256; do NMT_DEC_TILE=$t python tools/dec_gemm_sweep.py; done
