#!/bin/bash
# Re-measure the suite's tuned transforms on this GPU and rebuild the bundled
# facts file (run under gpurun): one fact per candidate, device b200.
#   bash tools/retune.sh [facts path]
DB=${1:-paper_2601_12220_b200/facts/b200.facts.new}
B=./paper_2601_12220_b200/bin/feinsum
rm -f "$DB"
$B tune tools/es/C1.es --db "$DB" --reps 20 --candidates "stages=2;ept=2;te=68,stages=1;ept=2;te=68,stages=4;ept=2,stages=3;ept=2,stages=4;te=16,stages=2;ept=2;te=64,stages=4"
$B tune tools/es/C5.fk --db "$DB" --reps 10 --candidates "stages=3;ept=2;te=64,stages=3;ept=2,stages=4;ept=2,stages=4;te=16"
$B tune tools/es/C2.es --db "$DB" --reps 3 --candidates ",ne=2,v=1"
$B tune tools/es/C3.fk --db "$DB" --reps 5 --candidates "stages=2;group=6,stages=2;group=12,stages=3;group=6,stages=3;group=12"
$B tune tools/es/C4-f64.es --db "$DB" --reps 10 --candidates ""
$B tune tools/es/C4-f32.es --db "$DB" --reps 10 --candidates ",tc=1"
$B tune tools/es/C1L-f32.es --db "$DB" --reps 10 --candidates "stages=4;ept=2;te=68,stages=4;ept=2,stages=3;ept=2,stages=3;ept=2;te=64,stages=4"
