#!/bin/bash
# Regenerates the round's measured artifacts on a B200 box (run under gpurun):
#   gpurun --timeout 1800 -- 'bash tools/round_artifacts.sh r01d'
# then, in the dev container:
#   bash tools/round_artifacts.sh r01d --summarize
# Outputs land in gpurun_out/<tag>_*; --summarize copies the judged summaries
# into profiles/.
TAG=${1:-rXX}
OUT=gpurun_out
summarize() {
  # the judged summaries of this run into $DEST (on the box: gpurun_out/<tag>_profiles,
  # merged back; the .ncu-rep files are too large to travel back all at once)
  DEST=$1
  mkdir -p $DEST
  for w in c3 c1 c2 c4 c5 ref; do
    [ -s $OUT/${TAG}_bench_$w.json ] && grep '^{' $OUT/${TAG}_bench_$w.json | tail -1 > $DEST/${TAG}_bench_$w.json
  done
  cp $OUT/${TAG}_launches.csv $DEST/${TAG}_launches.csv
  python tools/summarize_profiles.py launches $OUT/${TAG}_launches.csv > $DEST/${TAG}_launches_summary.txt
  python tools/summarize_profiles.py full $OUT/${TAG}_bp.ncu-rep \
    "$TAG: K1 N=1024 (c3 kernel), ncu --set full --clock-control none, tools/profile_kernels.py 16384 256 2.0" \
    > $DEST/${TAG}_ncu_bp.txt
  python tools/summarize_profiles.py full $OUT/${TAG}_bp4096.ncu-rep \
    "$TAG: K1 N=4096 (c4 kernel), tools/profile_kernels.py 2048 16 2.0 4096" > $DEST/${TAG}_ncu_bp4096.txt
  python tools/summarize_profiles.py full $OUT/${TAG}_bp128.ncu-rep \
    "$TAG: K1 N=128 (c1 kernel), tools/profile_kernels.py 65536 16 2.0 128" > $DEST/${TAG}_ncu_bp128.txt
  python tools/sass_mix.py $OUT/${TAG}_bp.ncu-rep 30 > $DEST/${TAG}_bp_sass_mix.txt
  python tools/summarize_profiles.py full $OUT/${TAG}_scl.ncu-rep \
    "$TAG: K3 N=1024 L=32 (c3 kernel), tools/profile_kernels.py 16 4096 1.5" > $DEST/${TAG}_ncu_scl.txt
  tail -3 $OUT/${TAG}_pytest.log > $DEST/${TAG}_pytest_gpu.txt
  python - "$OUT" "$TAG" "$DEST" <<'PY'
import csv, io, json, subprocess, sys
out, tag, dest = sys.argv[1], sys.argv[2], sys.argv[3]
def raw(rep):
    rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                      capture_output=True, text=True).stdout)))
    h, u, r = rows[0], rows[1], rows[2]
    def val(k):
        v = float(r[h.index(k)].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[h.index(k)], 1)
    return val, r[h.index("Kernel Name")]
issue = {}
for name, N, frames in (("bp", 1024, 16384), ("bp4096", 4096, 2048), ("bp128", 128, 65536)):
    rep = f"{out}/{tag}_{name}.ncu-rep"
    try:
        val, kern = raw(rep)
        it = int(open(f"{out}/{tag}_{name}.out").read().split("iterations")[1].split()[0])
    except Exception as e:
        print("skip", name, e)
        continue
    n = N.bit_length() - 1
    ipg = val("smsp__inst_executed.sum") / (it * 2 * n * N)
    issue[str(N)] = {"warp_inst_per_alg_g": ipg, "kernel": kern, "frames": frames, "iterations": it,
                     "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "xu_pct": val("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                     "source": f"profiles/{tag}_ncu_{name}.txt ({tag}_{name}.ncu-rep, smsp__inst_executed.sum / "
                               "(iterations x 2nN))"}
    if N == 1024:
        tot = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        json.dump({"kernel": kern, "frames_per_launch": frames, "dram_bytes_per_launch": tot,
                   "dram_bytes_per_frame": tot / frames, "algorithmic_bytes_per_frame": 4173,
                   "source": f"profiles/{tag}_ncu_bp.txt ({tag}_bp.ncu-rep)"},
                  open(dest + "/bp_kernel_ncu.json", "w"), indent=1)
json.dump(issue, open(dest + "/k1_issue.json", "w"), indent=1)
print(json.dumps(issue, indent=1))
PY
}
if [ "$2" == "--summarize" ]; then
  cp $OUT/${TAG}_profiles/* profiles/
  exit 0
fi
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/${TAG}_pytest.log 2>&1
tail -3 $OUT/${TAG}_pytest.log
timeout 400 python bench.py > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
timeout 400 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
for w in c1 c2 c4 c5; do
  timeout 400 python bench.py --workload $w > $OUT/${TAG}_bench_$w.json 2> $OUT/${TAG}_bench_$w.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_bp -c 1 -o $OUT/${TAG}_bp -f \
  python tools/profile_kernels.py 16384 256 2.0 > $OUT/${TAG}_bp.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_bp -c 1 -o $OUT/${TAG}_bp4096 -f \
  python tools/profile_kernels.py 2048 16 2.0 4096 > $OUT/${TAG}_bp4096.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_bp -c 1 -o $OUT/${TAG}_bp128 -f \
  python tools/profile_kernels.py 65536 16 2.0 128 > $OUT/${TAG}_bp128.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scl3 -c 1 -o $OUT/${TAG}_scl -f \
  python tools/profile_kernels.py 16 4096 1.5 > /dev/null 2>&1
ls -la $OUT | grep $TAG
for w in c3 ref c1 c2 c4 c5; do tail -c 400 $OUT/${TAG}_bench_$w.json; echo; done
summarize $OUT/${TAG}_profiles
# keep the K1 N=1024 report (for the source page); the others are summarized above
rm -f $OUT/${TAG}_bp4096.ncu-rep $OUT/${TAG}_bp128.ncu-rep $OUT/${TAG}_scl.ncu-rep
ls -la $OUT/${TAG}_profiles
