"""A/B per-pass timing of library builds on the same box, interleaved.

    python debug/ab.py libA.so libB.so [libC.so ...] [--reps 4] [--batch 64]

Each library is loaded in its own subprocess per repetition (ctypes cannot
unload), alternating A, B, A, B ... so clock/thermal drift hits all builds
alike.  Prints the mean and min per-pass ms for every build.
"""
import json, os, subprocess, sys

libs = [a for a in sys.argv[1:] if a.endswith('.so')]
reps = int(sys.argv[sys.argv.index('--reps') + 1]) if '--reps' in sys.argv else 4
batch = sys.argv[sys.argv.index('--batch') + 1] if '--batch' in sys.argv else '64'
res = {l: [] for l in libs}
for _ in range(reps):
    for l in libs:
        pr = subprocess.run([sys.executable, 'debug/passtime.py', batch, 'x'], capture_output=True, text=True,
                            env={**os.environ, 'HTB200_LIB': l}, timeout=300)
        if pr.returncode != 0:
            sys.exit(f"{l}: passtime failed\n{pr.stderr[-2000:]}")
        out = pr.stdout.strip().splitlines()[-1]
        d = eval(out.split(' ', 1)[1])
        res[l].append(d)
for l in libs:
    tags = sorted(res[l][0])
    mean = {t: round(sum(r[t] for r in res[l]) / len(res[l]), 4) for t in tags}
    mn = {t: round(min(r[t] for r in res[l]), 4) for t in tags}
    print(os.path.basename(l), 'mean', mean, 'min', mn)
