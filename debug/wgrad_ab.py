"""A/B of two library builds' 32->32 weight gradient (HTB200_LIB per subprocess)."""
import os, subprocess, sys
for lib in sys.argv[1:]:
    out = subprocess.run([sys.executable, "debug/wgrad_time.py"], capture_output=True, text=True,
                         env={**os.environ, "HTB200_LIB": lib}, timeout=300).stdout
    print(os.path.basename(lib), out.strip().replace("\n", " | "))
