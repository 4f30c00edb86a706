"""A/B of environment / flag variants through bench.py (each run a fresh
process; rounds alternate the variants, medians reported).

    python tools/ab_env.py rounds config 'NAME:ENV=V,ENV2=V2:flags[:budget]' ...
"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rounds, config, variants = int(sys.argv[1]), sys.argv[2], sys.argv[3:]
res = {v: [] for v in variants}
for _ in range(rounds):
    for v in variants:
        name, envs, flags, budget = (v.split(":") + ["", "", ""])[:4]
        env = dict(os.environ)
        for kv in filter(None, envs.split(",")):
            k, _, val = kv.partition("=")
            env[k] = val
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--no-cpu-baseline", "--steps", "20",
               "--warmup", "5", "--flags", flags or "0"] + (["--budget", budget] if budget else [])
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=ROOT)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            res[v].append(None)
            print(v, "ERR", out.stderr[-500:], flush=True)
            continue
        d = json.loads(line[-1])
        res[v].append(d["ms_per_step"] * 1e3)
        print(f"{v}: {d['ms_per_step'] * 1e3:.1f} us ok={d['verified']['ok']} budget={d['config'].get('tc_sm_budget')}",
              flush=True)
for v in variants:
    xs = [x for x in res[v] if x is not None]
    print(f"{config} {v:40s} median {statistics.median(xs):.1f} us  {['%.1f' % x for x in xs]}")
