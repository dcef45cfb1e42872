#!/bin/bash
# Run a command with a host-memory guard: kill it (SIGKILL) if the box's
# MemAvailable drops below $MEMGUARD_MIN_KB (default 16 GB), and log the
# minimum MemAvailable seen.  Usage: tools/memguard.sh <log> <cmd...>
log=$1; shift
min_kb=${MEMGUARD_MIN_KB:-16000000}
"$@" &
pid=$!
low=999999999999
while kill -0 $pid 2>/dev/null; do
  a=$(awk '/MemAvailable/{print $2}' /proc/meminfo)
  [ "$a" -lt "$low" ] && low=$a
  if [ "$a" -lt "$min_kb" ]; then
    echo "memguard: MemAvailable ${a} kB < ${min_kb} kB, killing $pid" >> "$log"
    kill -9 $pid
  fi
  sleep 1
done
wait $pid
rc=$?
echo "memguard: rc=$rc min MemAvailable ${low} kB" >> "$log"
exit $rc
