# scan_rda interval statistics (dev build) at C3, then the release build's timing
python -c "from paper_2602_23999_b200 import _build; _build.build(force=True, extra_flags=['-DIVRQ_RDA_STATS'] + '${EXTRA}'.split())" > gpurun_out/rda_build.log 2>&1 || tail gpurun_out/rda_build.log
IVRQ_KERNEL_TIMING=1 python tools/prof_search.py --config ${CFG:-c3} --nprobe ${NPROBE:-8} --reps 2 2>&1 | grep -E "rda|step ms|tc_|scan_" | tail -8
python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench, paper_2602_23999_b200 as iv
from paper_2602_23999_b200.index import build_index_device
cfg = bench.CONFIGS['c3']
x, q = bench.make_dataset_gpu(cfg['n'], 2000, cfg['d'], torch.device('cuda', 0))
ix = build_index_device(x, iv.BuildParams(n_clusters=cfg['nlist'], quant=iv.QuantizationParams(bits=cfg['bits']), kmeans_iters=25, train_fraction=bench.train_fraction(cfg['n'], cfg['nlist']), seed=0))
lf = ix.long_factors
print('long add: max %.4g  med %.4g | scale: max %.4g med %.4g p99.99 %.4g' % (np.abs(lf[:,0]).max(), np.median(np.abs(lf[:,0])), np.abs(lf[:,1]).max(), np.median(np.abs(lf[:,1])), np.quantile(np.abs(lf[:,1]), 0.9999)))
qh = q.cpu().numpy()
print('query |q| max per row: median %.4g' % np.median(np.abs(qh).max(1)))
PY
