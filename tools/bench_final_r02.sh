# final round-2 bench lines: cfg4 default (both arms), cfg0-cfg3
python bench.py > gpurun_out/bench_cfg4_r02.json 2> gpurun_out/bench_cfg4_r02.err; echo "cfg4 rc=$?"; tail -c 600 gpurun_out/bench_cfg4_r02.err
for c in 0 1 2 3; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg${c}_r02.json 2> gpurun_out/bench_cfg${c}_r02.err; echo "cfg$c rc=$?"; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_cfg4_r02.json 2> gpurun_out/bench_ref_cfg4_r02.err; echo "ref rc=$?"
python - <<'P'
import json
for c in (4,0,1,2,3):
    d=json.loads(open(f"gpurun_out/bench_cfg{c}_r02.json").read().strip().splitlines()[-1])
    print(c, d["ms_per_step"], d["value"], d["roofline"].get("tensor_pipe_frac"), d["roofline"].get("tensor_pipe_frac_step"), d["roofline"].get("traffic"), d.get("tts",{}).get("seconds"), d["clocks"])
P
