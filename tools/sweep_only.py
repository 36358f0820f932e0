import sys, json; sys.path.insert(0, ".")
import importlib.util
spec = importlib.util.spec_from_file_location("bench", "bench.py"); b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
from paper_1609_01689_b200 import ci
print(json.dumps(b.sweep_record(ci.Device(0))))
