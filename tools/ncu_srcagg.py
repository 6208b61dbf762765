import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; fname = None; out = []
for r in rows:
    if r and r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr[4:], r[4:]))
        try:
            out.append((fname, int(r[0]), r[1][:95], int(d['Instructions Executed'] or 0), int(d['Warp Stall Sampling (All Samples)'] or 0), float(d['Avg. Threads Executed'] or 0)))
        except Exception: pass
ti = sum(o[3] for o in out); ts = sum(o[4] for o in out)
print("total warp inst", ti)
for o in sorted(out, key=lambda o: -o[4])[:int(sys.argv[2])]:
    print(f"{100*o[3]/ti:5.1f}%i {100*o[4]/ts:5.1f}%s thr{o[5]:5.1f} {o[0]}:{o[1]} {o[2]}")
