import json, sys
for path in sys.argv[1:]:
    try:
        d = json.load(open(path))
    except Exception as e:
        print(path, "unreadable", e)
        continue
    print(path, "ms/frame", d["ms_per_step"], "e2e", d["e2e"]["ms_per_frame"], "outside", d.get("frame_ms_outside_stages"),
          "stages", d["stage_ms_per_frame"])
    for p, s in enumerate(d.get("stage_ms_per_pass_last_frame", [])):
        print("   pass", p, d["pass_stats"][p]["n_active_before"], s)
