"""Golden bytes of the reference's RGF1 / RPB1 containers (graph.py:219-290,
partition.py:97-119).  Runs in the build container only (imports gnnpipe
from /root/reference); writes tests/golden/golden_formats.json."""

import hashlib
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from gnnpipe.graph import save_graph, synth_powerlaw  # noqa: E402
from gnnpipe.partition import partition_edgecut, save_partition  # noqa: E402

out = {}
with tempfile.TemporaryDirectory() as d:
    for name, args in {"small": (1000, 5, 8, 4, 7), "tiny": (50, 3, 3, 2, 11)}.items():
        g = synth_powerlaw(*args)
        p = Path(d) / f"{name}.rgf"
        save_graph(g, p)
        b = p.read_bytes()
        q = Path(d) / f"{name}.rpb"
        save_partition(partition_edgecut(g, 2), q)
        c = q.read_bytes()
        out[name] = {"args": list(args), "rgf1_len": len(b),
                     "rgf1_blake2b": hashlib.blake2b(b, digest_size=16).hexdigest(),
                     "rpb1_len": len(c),
                     "rpb1_blake2b": hashlib.blake2b(c, digest_size=16).hexdigest()}
Path(__file__).with_name("golden_formats.json").write_text(json.dumps(out, indent=1))
print(out)
