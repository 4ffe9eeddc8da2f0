"""Steering-service host logic without a device (reference service.py:
138-221): message validation, the controller seat, acks, the session log
and grab release on disconnect, against a stub engine whose tickets resolve
immediately.  The GPU-backed protocol tests are in test_gpu_service.py."""

import json
import threading

import pytest

from paper_2509_04277_b200 import scenarios, service as svc_mod
from paper_2509_04277_b200.engine import Mailbox
from paper_2509_04277_b200.scene import build_world, parse_scene


class StubEngine:
    def __init__(self, world):
        self.world = world
        self.mailbox = Mailbox()
        self.posted = []

    def post_command(self, name, **args):
        ticket = self.mailbox.post(name, **args)
        self.posted.append((name, args))
        for _, t in self.mailbox.drain():
            t.resolve(self.world.step_index)
        return ticket


def make_service(tmp_path=None):
    cfg = parse_scene({"rods": [{"num_points": 24, "length": 0.2}]},
                      base_dir=scenarios.ASSET_DIR)
    s = svc_mod.SimService.__new__(svc_mod.SimService)
    s.config = cfg
    s.world = build_world(cfg)
    s.engine = StubEngine(s.world)
    s.batch, s.stride = cfg.batch, cfg.stream_stride
    s.session_log = None if tmp_path is None else str(tmp_path / "log.ndjson")
    s.controller, s.controller_grabs = None, set()
    s._lock = threading.Lock()
    s._params, s._thread, s.error = None, None, None
    s._stop = threading.Event()
    return s


def cmd(ident, kind, **args):
    return {"type": "command", "id": ident, "command": {"type": kind, **args}}


def reply(s, client, msg):
    return svc_mod._reply(s, client, msg if isinstance(msg, str) else json.dumps(msg))


def test_hello_scene_summary():
    s = make_service()
    h = s.hello()
    assert h["protocol_version"] == svc_mod.PROTOCOL_VERSION
    assert h["scene"]["rods"][0]["num_points"] == 24 and "mesh_url" not in h["scene"]


@pytest.mark.parametrize("msg,code,text", [
    ("{nope", "bad_json", ""),
    ({"type": "ping"}, "bad_message", ""),
    (cmd(1, "teleport"), "bad_command", "unknown command"),
    ({"type": "command", "id": 1, "command": {}}, "bad_command", "missing"),
    (cmd(1, "grab", index=99, target=[0, 0, 0]), "bad_command", "index out of range"),
    (cmd(1, "grab", index=3, target=[0, 0]), "bad_command", "grab target"),
    (cmd(1, "grab", index=3, rod=4, target=[0, 0, 0]), "bad_command", "rod index"),
    (cmd(1, "insert_velocity", value="fast"), "bad_command", "numeric"),
    (cmd(1, "set_params", gravity=1), "bad_command", "set_params accepts"),
    (cmd(1, "set_params"), "bad_command", "set_params accepts"),
])
def test_rejections(msg, code, text):
    r = reply(make_service(), 1, msg)
    assert r["type"] == "error" and r["code"] == code and text in r["message"]


def test_seat_acks_log_and_release_on_disconnect(tmp_path):
    s = make_service(tmp_path)
    s.world.step_index = 40
    a = reply(s, "alice", cmd(7, "grab", index=5, target=[0.0, 0.1, 0.0]))
    assert a == {"type": "ack", "id": 7, "apply_step": 40}
    assert reply(s, "bob", cmd(1, "rotate_velocity", value=1.0))["code"] == "controller_bound"
    assert s.controller_grabs == {(0, 5)}
    s.client_disconnected("bob")          # an observer leaving changes nothing
    assert s.controller == "alice"
    s.world.step_index = 60
    s.client_disconnected("alice")
    assert s.controller is None and s.controller_grabs == set()
    assert s.engine.posted[-1] == ("release", {"rod": 0, "index": 5})
    lines = [json.loads(x) for x in open(s.session_log).read().splitlines()]
    assert [(x["id"], x["step"], x["command"]["type"]) for x in lines] == [
        (7, 40, "grab"), (-1, 60, "release")]
    # the seat is free again
    assert reply(s, "bob", cmd(2, "rotate_velocity", value=0.0))["type"] == "ack"
    # the log is a replayable session
    assert [e[:2] for e in scenarios.load_replay(s.session_log)] == [
        (40, "grab"), (60, "release"), (60, "rotate_velocity")]
