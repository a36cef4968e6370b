import re, sys
t = open(sys.argv[1] if len(sys.argv) > 1 else 'paper_2009_10400_b200/lib/ptxas_summary.txt').read().split('Compiling entry function')
for b in t[1:]:
    name = re.search(r"'(\S+)'", b).group(1)
    regs = re.search(r'Used (\d+) registers', b).group(1)
    sp = re.search(r'(\d+) bytes spill stores', b).group(1)
    sl = re.search(r'(\d+) bytes spill loads', b).group(1)
    print(f'{regs:>4} regs spill {sp:>4}/{sl:>4}  {name[:60]}')
