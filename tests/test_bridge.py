"""Co-simulation bridge, protocol "tacchi/1".

The B200 bridge (csrc/bridge.cpp: Session + run_protocol over the device step
and capture path) is compared with the reference's own bridge::run_protocol
(server.cpp:49-113, session.cpp:15-98) run on the same script: golden replies,
steps.jsonl and .depth/.png outputs in tests/golden/bridge.npz
(tests/golden/make_golden.py::bridge). Protocol and config errors are host
logic and run on CPU; sessions that step need the GPU.

Tolerances for the stepped outputs are those of the capture parity tests
(tests/test_gpu_parity.py): depth <= 1e-7 m, image <= 2/255; the replies
(step, depth_m, terminal, paths) and steps.jsonl are exact.
"""
import json
import os
import socket
import subprocess
import threading

import numpy as np
import pytest

from tests.scenes import BAD_CONFIGS, SMALL, bridge_script

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SERVE = os.path.join(ROOT, "paper_2301_08343_b200", "_lib", "tacchi_serve")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "bridge.npz"))


def _tb():
    import paper_2301_08343_b200 as tb

    return tb


def test_config_errors_match_reference(golden, tmp_path):
    """init with an invalid SceneConfig -> PhysicsFault with the reference's
    ConfigError message (scene_config.cpp:83-116), session keeps serving."""
    tb = _tb()
    msgs = [{"type": "init", "config": c} for c in BAD_CONFIGS] + [{"type": "end"}]
    got = tb.bridge.run_protocol(msgs, session_root=str(tmp_path))
    assert got == json.loads(str(golden["bad_configs"]))


def test_protocol_errors_before_init(golden, tmp_path):
    tb = _tb()
    script = bridge_script(str(tmp_path / "s0"))
    got = tb.bridge.run_protocol(script[:2] + [{"type": "bogus"}, {"type": "end"}],
                                 session_root=str(tmp_path))
    ref = json.loads(str(golden["replies"]))
    assert got[:2] == ref[:2]
    assert got[2] == {"type": "error", "error": "ProtocolError",
                      "message": "unknown message type 'bogus'", "echo": '{"type": "bogus"}'}
    assert got[3] == {"type": "done", "steps": 0}


def test_serve_stdio_cli(tmp_path):
    """tools/tacchi_serve --stdio: newline-delimited JSON in, replies out."""
    if not os.path.exists(SERVE):
        pytest.skip("tacchi_serve not built")
    inp = "\n".join([json.dumps({"type": "init", "config": {"lights": []}}), "{", "",
                     json.dumps({"type": "end"}), json.dumps({"type": "init"})]) + "\n"
    p = subprocess.run([SERVE, "--root", str(tmp_path), "--stdio"], input=inp, text=True,
                       capture_output=True, timeout=60)
    assert p.returncode == 0, p.stderr
    lines = [json.loads(x) for x in p.stdout.splitlines()]
    assert [x["type"] for x in lines] == ["error", "error", "done"]  # stops at "end"
    assert lines[0]["message"] == "at least one light source required"
    assert lines[1]["message"] == "not valid JSON"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tcp_session(port, messages):
    import time

    for _ in range(200):
        try:
            c = socket.create_connection(("127.0.0.1", port), timeout=120)
            break
        except OSError:
            time.sleep(0.05)
    else:
        raise RuntimeError("bridge did not listen")
    with c:
        f = c.makefile("rw")
        out = []
        for m in messages:
            f.write(json.dumps(m) + "\n")
            f.flush()
            out.append(json.loads(f.readline()))
        return out


def test_serve_tcp(tmp_path):
    """serve_tcp (server.cpp:125-182): loopback, sequential connections."""
    tb = _tb()
    port = _free_port()
    th = threading.Thread(target=tb.bridge.serve,
                          kwargs=dict(session_root=str(tmp_path), port=port, max_connections=2))
    th.start()
    try:
        a = _tcp_session(port, [{"type": "init", "config": {"render": {"image_width": 1}}},
                                {"type": "step", "vector": [0, 0, 0]}, {"type": "end"}])
        b = _tcp_session(port, [{"type": "end"}])
    finally:
        th.join(timeout=60)
    assert a[0]["message"] == "render image size too small"
    assert a[1]["error"] == "SessionNotInitialized"
    assert a[2] == {"type": "done", "steps": 0} and b == [{"type": "done", "steps": 0}]
    assert not th.is_alive()


def _read_depth_bytes(raw):
    raw = bytes(raw)
    nl = raw.index(b"\n")
    return raw[:nl], np.frombuffer(raw[nl + 1:], dtype=np.float32)


@pytest.mark.gpu
def test_session_script_matches_reference(golden, tmp_path):
    """The full script: velocity / position commands, NonMonotonicTime, bad
    modes, image requests, terminal at max_depth_m and the frozen step after
    it — replies and steps.jsonl exact, outputs within capture tolerance."""
    tb = _tb()
    sdir = str(tmp_path / "s0")
    got = tb.bridge.run_protocol(bridge_script(sdir), session_root=str(tmp_path))
    ref = json.loads(str(golden["replies"]).replace("<dir>", sdir))
    assert got == ref
    with open(os.path.join(sdir, "steps.jsonl")) as f:
        assert f.read() == str(golden["steps_jsonl"]).replace("<dir>", sdir)
    imaged = {r["step"]: r for r in got if r.get("type") == "reply" and r["image"]}
    assert sorted(imaged) == [1, 3, 4]  # the frozen step repeats step 4's reply
    imaged = list(imaged.values())
    for r in imaged:
        k = r["step"]
        with open(r["depth_map"], "rb") as f:
            head, vals = _read_depth_bytes(f.read())
        ghead, gvals = _read_depth_bytes(golden[f"depth_{k}"])
        assert head == ghead
        np.testing.assert_allclose(vals, gvals, rtol=0, atol=1e-7)
        d, r_m = tb.load_depth_map(r["depth_map"])
        assert d.shape == (120, 160) and r_m == json.loads(head)["pixel_to_meter"]
        img = tb.load_png(r["image"])
        assert np.abs(img.astype(int) - golden[f"image_{k}"]).max() <= 2
    assert got[-1] == {"type": "done", "steps": 4}


@pytest.mark.gpu
def test_position_and_velocity_commands_agree(tmp_path):
    """A position trajectory p_k = k * v * dt_control drives the same motion as
    the velocity command v (session.cpp:79-89), up to the rounding of
    (p - offset) / dt_control."""
    tb = _tb()
    dtc = 2e-6 * 10
    v = -0.5
    depths = {}
    for mode in ("velocity", "position"):
        sdir = str(tmp_path / mode)
        msgs = [{"type": "init", "config": SMALL, "max_steps": 6, "session_dir": sdir}]
        for k in range(1, 7):
            vec = [0.0, 0.0, v] if mode == "velocity" else [0.0, 0.0, v * dtc * k]
            msgs.append({"type": "step", "mode": mode, "vector": vec, "request_image": k == 6})
        msgs.append({"type": "end"})
        out = tb.bridge.run_protocol(msgs, session_root=str(tmp_path))
        assert [m["step"] for m in out[1:7]] == list(range(1, 7))
        assert [m["terminal"] for m in out[1:7]] == [False] * 5 + [True]
        depths[mode] = (tb.load_depth_map(out[6]["depth_map"])[0], out[6]["depth_m"])
    np.testing.assert_allclose(depths["velocity"][1], depths["position"][1], rtol=1e-12)
    np.testing.assert_allclose(depths["velocity"][0], depths["position"][0], rtol=0, atol=1e-9)


@pytest.mark.gpu
def test_default_terminal_is_deepest_press_level(tmp_path):
    """Without max_depth_m / max_steps the session ends at the deepest
    press.depths_mm level (session.cpp:19-24)."""
    tb = _tb()
    cfg = dict(SMALL, press_grid={"depths_mm": [0.001, 0.003]})
    msgs = [{"type": "init", "config": cfg}]
    msgs += [{"type": "step", "vector": [0.0, 0.0, -0.5]} for _ in range(8)] + [{"type": "end"}]
    out = tb.bridge.run_protocol(msgs, session_root=str(tmp_path))
    terminal = [m["terminal"] for m in out[1:9]]
    # gap 0.02 mm + 3 um at 10 um per control step -> terminal after step 3
    assert terminal == [False, False, True] + [True] * 5
    assert [m["step"] for m in out[1:9]] == [1, 2, 3, 3, 3, 3, 3, 3]
    assert out[-1] == {"type": "done", "steps": 3}
    assert os.path.exists(os.path.join(out[0]["session_dir"], "steps.jsonl"))


@pytest.mark.gpu
def test_serve_tcp_session_matches_in_process(golden, tmp_path):
    """The same scripted session over loopback TCP (serve_tcp) gives the
    reference's replies, like the in-process transport."""
    tb = _tb()
    port = _free_port()
    sdir = str(tmp_path / "tcp")
    th = threading.Thread(target=tb.bridge.serve,
                          kwargs=dict(session_root=str(tmp_path), port=port, max_connections=1))
    th.start()
    try:
        script = [m for m in bridge_script(sdir) if not isinstance(m, str)]
        got = _tcp_session(port, script)
    finally:
        th.join(timeout=120)
    ref = [r for r in json.loads(str(golden["replies"]).replace("<dir>", sdir))
           if r.get("echo") != "not json"]
    assert got == ref
    assert not th.is_alive()
