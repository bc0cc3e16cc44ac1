import sys, re
lines = open(sys.argv[1]).read().splitlines()
cur = None
for i, l in enumerate(lines):
    m = re.search(r"Function properties for (\S+)", l)
    if m: cur = m.group(1)
    m2 = re.search(r"Used (\d+) registers", l)
    if m2 and cur and ('k_traceILb0ELb0' in cur or 'k_shade' in cur):
        print('  ', cur[8:22], m2.group(1), lines[i-1].strip())
