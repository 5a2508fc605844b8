# single-CTA threshold / shape A/B for small merge sorts (tools/small_sweep.py)
TAG=default python tools/small_sweep.py
TAG=k32 NSB_SMALL_K32=1 python tools/small_sweep.py
TAG=single8192 NSB_SINGLE_MAX=8192 python tools/small_sweep.py
TAG=single8192k32 NSB_SINGLE_MAX=8192 NSB_SMALL_K32=1 python tools/small_sweep.py
TAG=single4096k32 NSB_SINGLE_MAX=4096 NSB_SMALL_K32=1 python tools/small_sweep.py
TAG=single4096t4096 NSB_SINGLE_MAX=4096 NSB_TILE=4096 NSB_SMALL_K32=1 python tools/small_sweep.py
TAG=single2048t2048 NSB_SINGLE_MAX=2048 NSB_TILE=2048 python tools/small_sweep.py
TAG=single2048t1024 NSB_SINGLE_MAX=2048 NSB_TILE=1024 python tools/small_sweep.py
