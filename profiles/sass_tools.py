"""Extract one function's SASS from a .so (cuobjdump) and summarise its instruction mix."""
import collections
import re
import subprocess
import sys


def functions(so):
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*Function : ", txt)
    out = {}
    for p in parts[1:]:
        name = p.split("\n", 1)[0].strip()
        ins = [re.sub(r"\s*/\*[0-9a-fx]+\*/\s*$", "", l).strip() for l in p.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
        ins = [re.sub(r"^/\*[0-9a-f]+\*/\s*", "", i) for i in ins]
        out[name] = ins
    return out


if __name__ == "__main__":
    fs = functions(sys.argv[1])
    pat = sys.argv[2]
    for name, ins in fs.items():
        if re.search(pat, name):
            ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0] for i in ins if i)
            print(name, len(ins))
            print(ops.most_common(25))
            if len(sys.argv) > 3:
                for i in ins:
                    print("   ", i)
