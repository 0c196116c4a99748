"""Literal schedules at small orders / deep recursions (launch- and host-bound regime): time per
call with the current MK_LITERAL_STREAMS setting (TAG labels the line). Dev A/B tool."""
import json
import os
import sys

import torch

sys.path.insert(0, "tools")
import quick_gpu as q  # noqa: E402

res = {"tag": os.environ.get("TAG", "")}
for n, L in ((256, 2), (512, 2), (512, 3), (1024, 2), (1024, 3), (1024, 4), (2048, 2), (2048, 3), (2048, 4), (4096, 3), (4096, 4)):
    a = torch.randint(-8, 9, (n, n), device="cuda").double()
    b = torch.randint(-8, 9, (n, n), device="cuda").double()
    c = torch.empty_like(a)
    for algo, name in ((6, "ip"), (5, "tt")):
        a2, b2 = a.clone(), b.clone()
        ms = q.timeit(lambda: q.strassen(algo, a2, b2, c, L), reps=5, warm=2)
        res[f"{name}_n{n}_L{L}"] = round(ms, 3)
print(json.dumps(res), flush=True)
