#!/bin/bash
# ParaExp vs serial leapfrog on small grids: PARAEXP_NO_SMALL x PARAEXP_CONCURRENT (one B200)
echo "workload   no_small conc  paraexp_ms  serial_leapfrog_ms  speedup  launches"
for wl in ${WLS:-wave2d wave2d-5 wave2d-10 wave2d-20 wave2d-40 c1}; do
  for ns in 0 1; do for cc in 0 1; do
    PARAEXP_NO_SMALL=$ns PARAEXP_CONCURRENT=$cc timeout 300 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['paraexp']; print('%-10s %4s %6s %10.3f %14.3f %12.3f %8d' % ('$wl', $ns, $cc, d['ms_per_step'], p['serial_leapfrog_ms'], p['speedup_vs_serial_leapfrog'], d['gpu_launches']))"
  done; done
done
