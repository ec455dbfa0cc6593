"""Worker process of `_ddpool`: reads (key, (l, h, c, gamma, xi, m)) frames
on stdin, answers (key, ok, divided differences | error text) on stdout.
Imports only numpy / scipy (`_dense`), never torch or the CUDA library."""

import os
import pickle
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _dense import phi_divided_differences  # noqa: E402

_HDR = struct.Struct("<I")


def main():
    rd, wr = sys.stdin.buffer, sys.stdout.buffer
    while True:
        hdr = rd.read(_HDR.size)
        if len(hdr) < _HDR.size:
            return
        (size,) = _HDR.unpack(hdr)
        key, (l, h, c, gamma, xi, m) = pickle.loads(rd.read(size))
        try:
            out = (key, True, phi_divided_differences(l, h, c, gamma, xi, m))
        except Exception as exc:  # noqa: BLE001 - reported to the caller
            out = (key, False, f"{type(exc).__name__}: {exc}")
        blob = pickle.dumps(out, protocol=pickle.HIGHEST_PROTOCOL)
        wr.write(_HDR.pack(len(blob)) + blob)
        wr.flush()


if __name__ == "__main__":
    main()
