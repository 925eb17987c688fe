#!/bin/bash
# Build in-tree here (the .so files travel with the snapshot), then run the
# given command on a B200 through gpurun. Usage: scripts/gpu.sh TIMEOUT 'cmd'
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
