timeout 300 python tools/dbg_clusters.py 2>&1 | tail -6; timeout 300 python -m pytest tests/test_gpu_tensor.py -q -p no:cacheprovider -k "clusters or pruned" 2>&1 | tail -2
