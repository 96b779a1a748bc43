"""Count selected SASS opcodes of one kernel in a built library (offline check
before spending GPU time). argv: lib substring-of-mangled-name [opcode ...]"""
import subprocess, sys, re
lib, key = sys.argv[1], sys.argv[2]
ops = sys.argv[3:] or ["MOV", "F2FP", "FMNMX", "HADD2.F32", "S2R", "S2UR", "LDTM", "STTM", "UTCHMMA", "FFMA2", "FADD2"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, body = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); body[cur] = []
    elif cur and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
        body[cur].append(line)
for name, lines in body.items():
    if key in name:
        print(name[:100], "instructions:", len(lines))
        for op in ops:
            print(f"  {op:10s}", sum(1 for l in lines if re.search(r"\b" + re.escape(op) + r"\b", l)))
