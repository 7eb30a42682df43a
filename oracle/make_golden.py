"""Regenerates tests/golden/ref_kat.json from the reference's own rng.hpp /
quaternion.hpp (compiled in place by oracle/Makefile.ref).  Run in a container
that has /root/reference; the JSON is committed so tests never need it."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "ref_kat.json")

if __name__ == "__main__":
    subprocess.run(["make", "-s", "-C", HERE, "-f", "Makefile.ref"], check=True)
    txt = subprocess.run([os.path.join(HERE, "_ref", "ref_kat")], check=True, capture_output=True,
                         text=True).stdout
    import json
    json.loads(txt)  # validate
    with open(OUT, "w") as f:
        f.write(txt)
    print("wrote", OUT)
