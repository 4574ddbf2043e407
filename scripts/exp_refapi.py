"""bench.reference_api_legs on its own (HydroSim + driver through the
mirrored reference API, native engine), printed as JSON."""
import json
import sys
import types

sys.path.insert(0, ".")
sys.argv = ["bench.py"]
import bench  # noqa: E402

if __name__ == "__main__":
    args = types.SimpleNamespace(no_cpu_baseline="--no-cpu" in sys.argv[1:])
    print(json.dumps(bench.reference_api_legs(args)))
