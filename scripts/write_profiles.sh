#!/bin/bash
# Copy one evidence run (scripts/gpu_profile_r02.sh TAG + the probes and the
# reference arm run after it, outputs in gpurun_out/) into the tracked
# round-2 summaries under profiles/.
#   scripts/write_profiles.sh r02s5
set -e
cd "$(dirname $0)/.."
T=gpurun_out/$1
grep '^{' ${T}_bench.log | tail -1 > profiles/r02_bench_latest.jsonl
for w in cfg4 cfg5-pcisph cfg5-wcsph; do grep '^{' ${T}_wl_$w.log | tail -1 >> profiles/r02_bench_latest.jsonl; done
grep '^{' ${T}_ref.log | tail -1 > profiles/r02_reference_arm.jsonl
(echo "# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-wcsph --no-e2e (cfg2 1M RTS-PCISPH; the graph-mode timed majors are not profilable -- conditional nodes -- so the list shows the host-driven instrumented pass: same kernels, launched one by one; cold caches, serialised)"; python scripts/launch_summary.py ${T}_launches.csv) > profiles/r02_pcisph_launches.txt
cp ${T}_launches.csv profiles/r02_pcisph_launches.csv
(echo "# ncu launch list: python bench.py --workload cfg5-wcsph --steps 1 --warmup 1 (4M RTS-WCSPH; one step graph per base step)"; python scripts/launch_summary.py ${T}_wcsph_launches.csv) > profiles/r02_wcsph_launches.txt
python scripts/make_traffic.py ${T}_traffic.csv > profiles/ncu_traffic.json
cp ${T}_traffic.csv profiles/r02_ncu_traffic_pcisph.csv
(echo "# ncu --set full --import-source on --clock-control none -k regex:'k_density|k_pforces' -c 2 (first launches: full pred / force sets, 1M); summary + hottest SASS by warp-stall samples"; python scripts/ncu_summary.py ${T}_full_pair.ncu-rep; python scripts/ncu_hot.py ${T}_full_pair.ncu-rep 12) > profiles/r02_ncu_pair_full.txt
(echo "# ncu --set full --import-source on --clock-control none -k regex:k_refresh\$ -s 3 -c 1 python scripts/refresh_probe.py 2 (the full refresh at a major start, 1M, SoA copies fresh); summary, then stall samples / warp instructions / active lanes per CUDA source line (scripts/ncu_lines.py)"; python scripts/ncu_summary.py ${T}_refresh_probe_full.ncu-rep; python scripts/ncu_lines.py ${T}_refresh_probe_full.ncu-rep k_refresh 30) > profiles/r02_ncu_refresh_full.txt
(echo "# scripts/refresh_probe.py 20 and scripts/graph_phase_probe.py 20 3 (cfg2 1M, warm, CUDA events / in-graph %globaltimer stamps)"; cat ${T}_refresh_probe.log ${T}_graph_phase.log) > profiles/r02_refresh_and_phases.txt
cp ${T}_refresh_probe_full.ncu-rep profiles/r02_refresh_full.ncu-rep
cp ${T}_full_pair.ncu-rep profiles/r02_pair_full.ncu-rep
echo "profiles written from $T"
