import csv, collections, re, sys, json
def load(path):
    lines=open(path).read().splitlines()
    start=next(i for i,l in enumerate(lines) if l.startswith('"ID"'))
    rows=list(csv.reader(lines[start:]))
    h=rows[0]; data=[r for r in rows[1:] if len(r)==len(h)]
    ix={n:i for i,n in enumerate(h)}
    agg=collections.OrderedDict()
    for r in data:
        k=(int(r[ix["ID"]]), r[ix["Kernel Name"]])
        agg.setdefault(k,{})[r[ix["Metric Name"]]]=(float(r[ix["Metric Value"]].replace(",","")), r[ix["Metric Unit"]])
    out=[]
    for (i,name),m in agg.items():
        short=re.sub(r"\(.*","",name).replace("void ","").replace("<unnamed>::","")
        def tob(v): return v[0]*{"byte":1,"Kbyte":1e3,"Mbyte":1e6,"Gbyte":1e9,"B":1,"KB":1e3,"MB":1e6,"GB":1e9}[v[1]]
        def tous(v): return v[0]*{"nsecond":1e-3,"usecond":1,"msecond":1e3,"ns":1e-3,"us":1,"ms":1e3}[v[1]]
        out.append((i, short, tous(m["gpu__time_duration.sum"]), tob(m["dram__bytes_read.sum"]), tob(m["dram__bytes_write.sum"])))
    return out
if __name__ == "__main__":
    for w in sys.argv[1:]:
        L=load(f"gpurun_out/launches_{w}.csv")
        by=collections.OrderedDict()
        for i,s,t,rd,wr in L: by.setdefault(s,[]).append((t,rd+wr))
        print("==",w, "launches", len(L))
        for k,v in by.items():
            print(f"  {k[:72]:72s} n={len(v):3d} us={sum(a for a,b in v)/len(v):9.1f} MB={sum(b for a,b in v)/len(v)/1e6:9.1f}")
