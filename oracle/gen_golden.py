"""Regenerate tests/golden/rng_kat.json from the REFERENCE header.

Runs oracle/_ref/rng_kat, which `make -C oracle ref` compiles from
/root/reference/proj/include/frag/common.hpp (the reference's own Rng,
common.hpp:45-100). Only runnable in the build container (the GPU box has no
/root/reference); the committed fixture is what tests read. Test
infrastructure only.
"""
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE.parent / "tests" / "golden" / "rng_kat.json"


def main():
    subprocess.run(["make", "-C", str(HERE), "ref"], check=True)
    txt = subprocess.run([str(HERE / "_ref" / "rng_kat")], check=True, capture_output=True, text=True).stdout
    data = json.loads(txt)
    payload = {"source": "/root/reference/proj/include/frag/common.hpp:45-100 via oracle/_ref/rng_kat",
               "generator": "oracle/gen_golden.py", "vectors": data}
    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(payload, indent=1) + "\n")
    print(f"wrote {OUT} ({len(data)} seeds)")


if __name__ == "__main__":
    sys.exit(main())
