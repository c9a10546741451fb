KGC_BUILD_EXPERIMENTS=1 python -c "from paper_2307_12059_b200 import _build; _build.build(force=True)" > gpurun_out/b.log 2>&1 || { tail gpurun_out/b.log; exit 1; }
for L in 1 2 4 8; do
  echo "LPC $L"
  KGC_VERIFY_LPC=$L timeout 300 python scripts/engine_ab.py c4 2 1e-5 'pivots=8' 2>&1 | tail -1 | grep -o '"ms_recheck": [0-9.]*'
  KGC_VERIFY_LPC=$L timeout 300 python scripts/engine_ab.py c2 2 1e-4 'pivots=8' 2>&1 | tail -1 | grep -o '"ms_recheck": [0-9.]*'
  KGC_VERIFY_LPC=$L timeout 300 python scripts/engine_ab.py c2 1 1e-4 'pivots=8' 2>&1 | tail -1 | grep -o '"ms_recheck": [0-9.]*'
  KGC_VERIFY_LPC=$L timeout 300 python scripts/engine_ab.py c3 2 1e-4 'pivots=1' 2>&1 | tail -1 | grep -o '"ms_recheck": [0-9.]*'
done
for K in 0 1; do echo "KD $K"; KGC_KD=$K timeout 300 python scripts/engine_ab.py c4 2 1e-5 'pivots=8' 2>&1 | tail -1 | cut -c1-330; done
