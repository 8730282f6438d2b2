BM_TRACE=3 python tools/step_var2.py c3_e8 10 > gpurun_out/stepvar5.log 2>&1; grep -E "^step" gpurun_out/stepvar5.log
python - <<'PY'
import re
cur=[]; out=[]
for line in open("gpurun_out/stepvar5.log"):
    if line.startswith("[bm trace host]"):
        cur.append(line.strip())
    elif line.startswith("step"):
        tot=float(line.split()[1])
        if tot > 260: out.append((line.strip(), cur))
        cur=[]
for st, c in out[:3]:
    print(st)
    for l in c:
        v=float(l.split()[-2])
        if v > 2: print("   ", l)
PY
