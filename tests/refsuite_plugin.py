"""pytest plugin: run the REFERENCE's own runtime / daemon / acceptance test
files, unmodified, against this package's GPU worker and GPU memory daemon.

Loaded with `-p refsuite_plugin` by tests/test_gpu_reference_suites.py. It
changes nothing in the reference's tests or package; it only re-targets the
two process roles the frozen seam lets a backend replace:

* `elastencil.launcher._spawn` (launcher.py:45-56) keeps spawning the
  reference coordinator (`elastencil.cli _coordinator`) but starts
  `paper_2512_19851_b200.worker` for the `_worker` role and
  `paper_2512_19851_b200.daemon` for the `_daemon` role, with the same
  arguments (`--id`, `--coordinator`, `--scratch`);
* `elastencil.daemon.MemoryDaemon` (used in-process by test_daemon.py) is
  `GpuMemoryDaemon`, so the reference `DaemonClient` talks to the GPU daemon
  over the reference daemon protocol.
"""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

ROLES = {"_worker": "paper_2512_19851_b200.worker", "_daemon": "paper_2512_19851_b200.daemon"}


def pytest_configure(config):
    for p in (REF, ROOT):
        if p not in sys.path:
            sys.path.insert(0, p)
    # spawned processes (coordinator: reference; workers / daemons: GPU) see both trees
    os.environ["PYTHONPATH"] = os.pathsep.join([ROOT, REF, os.environ.get("PYTHONPATH", "")])

    import elastencil.daemon as ref_daemon
    import elastencil.launcher as ref_launcher

    from elastencil.errors import SpawnFailed

    from paper_2512_19851_b200.daemon import GpuMemoryDaemon

    original = ref_launcher._spawn

    def _spawn(args, log_path):
        module = ROLES.get(args[0])
        if module is None:
            return original(args, log_path)
        log_file = open(log_path, "ab")
        try:
            return subprocess.Popen([sys.executable, "-m", module, *args[1:]], stdout=log_file,
                                    stderr=log_file, start_new_session=True)
        except OSError as exc:
            raise SpawnFailed(str(exc))

    ref_launcher._spawn = _spawn
    ref_daemon.MemoryDaemon = GpuMemoryDaemon
